"""Whole-network parity against the reference package itself.

For a network workload (cfg1 / cfg2 / cfg4; cfg3 is ~12 core-hours in the
reference) this encrypts the seeded inputs and evaluates the whole network
twice on the same host:

  * on the GPU through the public API (engine.encrypt_tensor_batched +
    engine.eval_encrypted, batched encoding);
  * with the reference `hecnet` from baseline/_ref (its own keygen,
    fv.encrypt in the same RNG draw order, and the engine.eval_encrypted
    loop with constant plaintexts over a fork pool; refarm.full_pass),

and compares the SHA-256 of the output ciphertext bodies ([B][2][k][n]
u64): equal digests mean every output ciphertext is bit-identical.

usage: python tools/fullpass_parity.py cfg2 [--out profiles/fullpass_cfg2.json]
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import refarm  # noqa: E402


def gpu_digest(workload: str):
    import torch

    import bench
    from paper_1811_09953_b200 import engine

    W, P, sk, pk, ek, net, cfg, x, tensor = bench._setup(workload)
    comp = engine.compile_network(net, cfg)
    t0 = time.perf_counter()
    out = engine.eval_encrypted(comp, tensor, ek, cfg, encoding="batched")[0]
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    return {"out_sha256": refarm.output_digest(out.buf), "in_sha256": refarm.output_digest(tensor.buf),
            "eval_s_first_call": t, "out_scale": out.scale_exponent, "outputs": int(out.buf.shape[0])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=["cfg1", "cfg2", "cfg4"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--cores", type=int, default=None)
    args = ap.parse_args()
    g = gpu_digest(args.workload)
    print(f"[parity] gpu {args.workload}: {g}", flush=True)
    r = refarm.full_pass(args.workload, args.cores, log=lambda m: print(m, flush=True))
    res = {"workload": args.workload, "gpu": g, "reference": r,
           "bit_identical": g["out_sha256"] == r["out_sha256"] and g["out_scale"] == r["out_scale"]}
    line = json.dumps(res)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
