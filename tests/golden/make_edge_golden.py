"""Run the reference (/root/reference, importable in the build container only) on the
edge-case listings of edge_listings.py and write tests/golden/edge.json: for each
listing, config and seed, the sha256 of anneal(...).history_jsonl() and the best /
current schedules as permutations of the input order.

    python tests/golden/make_edge_golden.py
"""
import hashlib
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))

import sasstune as ref  # noqa: E402

from edge_listings import EDGE_LISTINGS  # noqa: E402
from golden_configs import CONFIGS  # noqa: E402

SEEDS = range(32)
CFGS = ("default", "unsafe", "long")


def perm_of(kernel, schedule) -> list:
    index = {id(ins): i for i, ins in enumerate(kernel.schedule)}
    return [index[id(ins)] for ins in schedule]


def main() -> None:
    out = {}
    for name, text in sorted(EDGE_LISTINGS.items()):
        k = ref.parse_kernel(text, name=name)
        rec = {"text": text, "anneal": {}}
        for cname in CFGS:
            runs = {}
            for s in SEEDS:
                st = ref.anneal(k, ref.SimulatorBackend(), ref.AnnealConfig(seed=s, **CONFIGS[cname]))
                runs[str(s)] = {"sha256": hashlib.sha256(st.history_jsonl().encode()).hexdigest(),
                                "best": perm_of(k, st.best.schedule),
                                "current": perm_of(k, st.current.schedule)}
            rec["anneal"][cname] = runs
        out[name] = rec
    (HERE / "edge.json").write_text(json.dumps(out, indent=0, sort_keys=True) + "\n")
    print("wrote", HERE / "edge.json")


if __name__ == "__main__":
    main()
