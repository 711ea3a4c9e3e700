"""cfg5 primitive pass (BASELINE.json configs[4]) and its multi-GPU split.

The workload: N = 16384, 8 limbs of ~50 bits,
beta = 2^134 ("dnum = 3": ell + 1 = 3 key-switching digits), a batch of
4,096 uniform ciphertexts, and three primitives of the evaluation path:

  * forward + inverse NTT of every polynomial (reference ring.py:242-255),
  * ciphertext square + relinearisation (fv.mul_ct(x, x), fv.py:498-549),
  * a 1024-term sparse power-of-two scalar MAC: 4,096 outputs, each the sum
    of 1,024 signed 2^e multiples (e in [0, 6]) of distinct inputs -- a
    linear layer of the reference evaluator (engine.py:698-717).

One pass chains them like a network stage: the NTT round trip runs on the
rank's ciphertexts, the squares are the MAC's inputs.  Multi-GPU split
(SURVEY 8(e)): the NTT and the square + relinearisation are pure ciphertext
sharding (contiguous blocks, no exchange); the MAC needs every input, so the
squares are all-gathered once (NCCL over NVLink), and its output rows are
partitioned the same way.  `primitive_schedule` holds that schedule apart
from the compute, which the CPU (gloo) tests run with the oracle.
"""

from __future__ import annotations

from .dist import partition


def primitive_schedule(x_local, rank: int, world: int, count: int, n_out: int, ntt_roundtrip, square, gather,
                       mac_rows):
    """The sharded pass over this rank's block of the `count` ciphertexts.

    ntt_roundtrip(x_local) -> NTT fwd+inv of the block
    square(x_local)        -> relinearised squares of the block
    gather(local, count, block) -> all `count` squares on every rank
    mac_rows(full, lo, hi) -> MAC outputs [lo, hi) of `n_out`
    Returns (ntt block, square block, MAC block)."""
    parts = partition(count, world)
    block = parts[0][1] - parts[0][0]
    nt = ntt_roundtrip(x_local)
    sq = square(x_local)
    full = gather(sq, count, block)
    lo, hi = partition(n_out, world)[rank]
    mac = mac_rows(full, lo, hi)
    return nt, sq, mac


class PrimitivePass:
    """The cfg5 pass on this rank's GPU (one process per GPU).

    `run(x_local)` executes primitive_schedule with the libfcn kernels and
    records CUDA events around each primitive (`times()` after a sync)."""

    def __init__(self, params, ek, plan, rank: int = 0, world: int = 1, group=None, chunk: int = 256):
        import torch

        from . import engine, fv

        self.P, self.ek, self.plan = params, ek, plan
        self.rank, self.world, self.group = rank, world, group
        self.count = max(max(tp.in_index for tp in o.taps) for o in plan.outputs if o.taps) + 1
        self.n_out = len(plan.outputs)
        t = int(params.t_lanes[0])
        self.low = engine._lower_linear(plan, t, params.n, "batched")
        lo, hi = partition(self.count, world)[rank]
        self.block = (lo, hi)
        self.ws = fv.mul_ct_workspace(params, max(1, min(chunk, hi - lo)))
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        self.nt_buf = None

    def _ntt(self, x_local):
        from . import _lib
        from . import device as dev

        h = self.P.native()
        k = len(self.P.limb_primes)
        if self.nt_buf is None or self.nt_buf.shape != x_local.shape:
            self.nt_buf = x_local.clone()
        else:
            self.nt_buf.copy_(x_local)
        rows = x_local.shape[0] * 2 * k
        L = _lib.lib()
        if rows:
            _lib.check(L.fcn_ntt_forward(h.ring_ptr, self.nt_buf.data_ptr(), rows, k, 0, dev.stream_ptr()))
            _lib.check(L.fcn_ntt_inverse(h.ring_ptr, self.nt_buf.data_ptr(), rows, k, 0, dev.stream_ptr()))
        return self.nt_buf

    def run(self, x_local):
        from . import dist as fdist
        from . import engine, fv

        ev = self.events
        P, ek = self.P, self.ek

        def ntt(x):
            ev[0].record()
            out = self._ntt(x)
            ev[1].record()
            return out

        def square(x):
            out = fv.mul_ct_batch(P, ek, 0, x, None, workspace=self.ws) if x.shape[0] else x.clone()
            ev[2].record()
            return out

        def gather(local, count, block):
            if self.world == 1:
                full = local
            else:
                full = fdist._torch_gather(local, count, block, self.group)
            ev[3].record()
            return full

        def mac_rows(full, lo, hi):
            lw = ("linear", self.low[0], self.low[1])
            out = engine._layer_range(P, 0, ek, self.plan, lw, full, lo, hi, "batched") if hi > lo else full[:0].clone()
            ev[4].record()
            return out

        return primitive_schedule(x_local, self.rank, self.world, self.count, self.n_out, ntt, square, gather,
                                  mac_rows)

    def times(self) -> dict:
        """Seconds of the last run's primitives (call after synchronising)."""
        ev = self.events
        return {
            "ntt_fwd_inv_s": ev[0].elapsed_time(ev[1]) / 1e3,
            "square_relin_s": ev[1].elapsed_time(ev[2]) / 1e3,
            "allgather_s": ev[2].elapsed_time(ev[3]) / 1e3,
            "mac_s": ev[3].elapsed_time(ev[4]) / 1e3,
        }


def uniform_batch(params, count: int, seed: int = 0, device=None):
    """`count` uniform ciphertexts [count][2][k][n] drawn on the GPU from a
    seeded generator (every rank draws the same batch and keeps its block)."""
    import torch

    k = len(params.limb_primes)
    g = torch.Generator(device=device or "cuda").manual_seed(seed)
    qs = torch.tensor(list(params.limb_primes), dtype=torch.int64, device=device or "cuda").view(1, 1, k, 1)
    x = torch.randint(0, 1 << 62, (count, 2, k, params.n), device=device or "cuda", generator=g, dtype=torch.int64)
    return (x % qs).contiguous()
