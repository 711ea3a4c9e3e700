"""cfg5 primitive throughput sweep (BASELINE.json configs[4]).

N=16384, 8 x ~50-bit limbs, 4096 random uniform ciphertexts (seed 0):
  * forward + inverse NTT of all 8192 polynomials,
  * ciphertext square + relinearisation with a dnum=3 key (beta = 2^134),
  * 1024-term sparse power-of-two MAC: 4096 outputs over the 4096 inputs.
Prints one JSON line (per-op times, GB/s vs the HBM copy peak, the NTT's
butterflies/s vs the measured FP64 butterfly peak, the key-switching inner
product's GB/s); optionally writes it to a file.

usage: python tools/sweep.py [--out profiles/sweep_r01.json] [--count 4096]
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_09953_b200 import _lib, configs, engine, fv  # noqa: E402
from paper_1811_09953_b200 import device as dev  # noqa: E402


def timed(fn, iters=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--mac-terms", type=int, default=1024)
    args = ap.parse_args()
    W = configs.WORKLOADS["cfg5"]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    k, n, B = len(W.primes), W.n, args.count
    h = P.native()
    sk, pk, ek = fv.keygen(P, configs.SEED_KEYS)
    g = torch.Generator(device="cuda").manual_seed(0)
    # random uniform residues per limb (device RNG; the workload is timing-only here)
    qs = torch.tensor(list(W.primes), dtype=torch.int64, device="cuda").view(1, 1, k, 1)
    x = (torch.randint(0, 1 << 62, (B, 2, k, n), device="cuda", generator=g, dtype=torch.int64) % qs).contiguous()
    ct_bytes = 2 * k * n * 8
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    fp = json.load(open(os.path.join(REPO, "profiles", "fp64_peak.json")))
    L = _lib.lib()
    st = dev.stream_ptr()
    res = {"workload": "cfg5", "n": n, "limbs": k, "ciphertexts": B, "beta_log2": 134, "dnum": P.ell + 1}

    # NTT forward + inverse over all 2B polys
    y = x.clone()

    def ntt():
        _lib.check(L.fcn_ntt_forward(h.ring_ptr, y.data_ptr(), 2 * B * k, k, 0, st))
        _lib.check(L.fcn_ntt_inverse(h.ring_ptr, y.data_ptr(), 2 * B * k, k, 0, st))

    t = timed(ntt)
    byts = 4 * B * ct_bytes  # read+write, both directions
    bfly = 2 * (2 * B * k) * (n // 2) * (n.bit_length() - 1)
    res["ntt_fwd_inv_s"] = t
    res["ntt_gbs"] = byts / t / 1e9
    res["ntt_frac_hbm"] = byts / t / 1e9 / peak
    rs = L.fcn_ntt_f64_schedule(n.bit_length() - 1, max(W.primes))
    res["ntt_fp64_schedule"] = rs
    res["ntt_frac_fp64_butterfly_peak"] = bfly / t / (fp.get("butterfly_rs1_per_s", fp["butterfly_per_s"])
                                                       if rs >= 1 else fp["butterfly_per_s"])
    assert torch.equal(y, x)

    # square + relinearisation (dnum = 3)
    ws = fv.mul_ct_workspace(P, 256)
    out = dev.empty(x.shape)

    def sq():
        fv.mul_ct_batch(P, ek, 0, x, None, out=out, workspace=ws)

    t = timed(sq, iters=2)
    byts = 2 * B * ct_bytes + 2 * (P.ell + 1) * k * n * 8  # in + out + keys once
    res["square_relin_s"] = t
    res["square_relin_gbs"] = byts / t / 1e9
    res["square_relin_frac_hbm"] = byts / t / 1e9 / peak
    res["square_relin_cts_per_s"] = B / t
    K = len(W.primes) + len(h.aux)
    rows = 2 * K + 3 * K + (P.ell + 1) * k + 2 * k  # NTT rows per square (fused fwd, tensor INTT, digits, final INTT)
    res["square_relin_ntt_rows_per_ct"] = rows
    res["square_relin_note"] = (
        f"FP64-bound, not HBM-bound: each square runs {rows} NTT rows of n={n} over the {K}-limb extended base "
        "plus the exact rescale; square_relin_frac_hbm only relates the in/out/key bytes (SURVEY 8(d)) to the time")

    # key-switching inner product alone (digits -> accumulators), 256 cts per launch
    D = P.ell + 1
    dig = (torch.randint(0, 1 << 62, (256, D, k, n), device="cuda", generator=g, dtype=torch.int64)
           % qs.view(1, 1, k, 1)).contiguous()
    acc = torch.empty((256, 2, k, n), device="cuda", dtype=torch.int64)
    kh = ek.native(P)

    def km():
        _lib.check(L.fcn_key_mac(h.ptr, kh.ptr, dig.data_ptr(), acc.data_ptr(), 256, st))

    t = timed(km, iters=10)
    res["keymac_s_per_256"] = t
    res["keymac_gbs"] = 256 * (D * k + 2 * k) * n * 8 / t / 1e9
    res["keymac_frac_hbm"] = res["keymac_gbs"] / peak

    # 1024-term sparse pow2 MAC, 4096 outputs over the 4096 inputs
    plan = configs.mac_sweep_plan(n_out=B, n_in=B, terms=args.mac_terms, seed=1)
    mac, _, _ = engine._lower_linear(plan, W.t, n, "batched")

    def macf():
        engine._mac_out(P, mac, x, None)

    t = timed(macf, iters=1)
    term_coeffs = B * args.mac_terms * 2 * k * n
    res["mac_s"] = t
    res["mac_term_coeffs_per_s"] = term_coeffs / t
    res["mac_gbs_algorithmic"] = 2 * B * ct_bytes / t / 1e9
    res["mac_l2_read_gbs"] = term_coeffs * 8 / t / 1e9
    res["fallbacks"] = h.fallbacks()
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
