# e2e overhead profile: SlotRow vs dense rows
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/e2e_profile.py 265216 > gpurun_out/r2o_e2e_slots.log 2>&1
SIP_NO_SLOTS=1 timeout 600 python tools/e2e_profile.py 227328 > gpurun_out/r2o_e2e_dense.log 2>&1
timeout 600 nsys --version > /dev/null 2>&1 || true
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2o_e2e_launches.csv python tools/e2e_profile.py 265216 > /dev/null 2>&1
