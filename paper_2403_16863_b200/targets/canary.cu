// canary.cu -- proves on hardware that a patched .text is what executes:
// exchanging the FFMA with the STG that stores its result must change y.
extern "C" __global__ void canary_axpy(const float* __restrict__ x, float* __restrict__ y, float a, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * x[i] + y[i];
}
