"""Per-stage times of square + relinearisation at a workload's shape
(fcn_stage_timing CUDA events; bench._square_relin_stages).

usage: [FCN_LIB_PATH=abvar/X/libfcn.so] python tools/stagebench.py [workload] [count]
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
from paper_1811_09953_b200 import configs, fv  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    W = configs.WORKLOADS[wl]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = fv.keygen(P, configs.SEED_KEYS)
    total, st = bench._square_relin_stages(P, ek, count, iters=5)
    print(json.dumps({"workload": wl, "count": count, "lib": os.environ.get("FCN_LIB_PATH", "default"),
                      "total_ms": total * 1e3, "stage_ms": {k: v * 1e3 for k, v in st.items()}}))


if __name__ == "__main__":
    main()
