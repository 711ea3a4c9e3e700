"""Host side of the tensor-core linear layer (csrc/mac_tc.cu, fcn_linear_mac_tc).

A linear layer of the reference evaluator (engine.py:698-717) is, in the
SIMD-batched encoding, out[o] = sum_t c_ot in[i_t] with small signed integer
constants c (|c| <= 64 for the workloads' power-of-two weights).  Lowered for
the tensor cores it becomes a set of dense int8 tiles:

  * output groups of up to 128 rows; each group's K list is the union of the
    inputs its rows read, and its weights are a dense int8 matrix over that
    list (zeros for pruned terms), pre-laid-out in the K-major canonical
    shared-memory layout the kernel copies with one bulk (TMA) transfer per
    64-input chunk;
  * the grouping is chosen among "positions" splits: outputs o = c S + s (S
    outputs per channel; a convolution's spatial positions), grouping every
    channel of a few consecutive positions so the K list is the union of a
    few receptive fields; S = n_out is the plain dense split (consecutive
    outputs).  A cost model (seconds on B200) picks the
    split and decides between this kernel and the sparse CUDA-core kernel
    (mac_fast_kernel); FCN_MAC_TC=0 / 1 forces the sparse / tensor-core path.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as dev

TILE_M, CHUNK, TILE_N = 128, 64, 64
TILE_BYTES = TILE_M * CHUNK

# B200 cost model, fitted to tools/macbench.py (profiles/r02_macbench.json):
T_CHUNK = 1.17e-6   # s per (64-input chunk x 64-column tile) on one SM (P = 7 planes)
T_TILE = 2.0e-6     # s per tile on one SM (accumulator drain, store, pipeline turn-around)
N_SM = 148
R_HBM = 5.5e12      # bytes/s streamed (byte-plane split: 8 + P bytes per residue)
R_SPARSE = 2.1e12   # term-coefficients/s of mac_fast_kernel
R_SPARSE_IO = 3.0e12  # bytes/s of its input + output traffic


@dataclass
class TcPlan:
    groups: object  # device int32 [G][8]
    kidx: object    # device int32
    rows: object    # device int32
    wimg: object    # device int8
    n_groups: int
    n_out: int
    split: int      # outputs per channel S of the chosen grouping
    est_tc: float
    est_sparse: float


def _mode() -> str:
    v = os.environ.get("FCN_MAC_TC", "auto")
    return {"0": "off", "1": "on"}.get(v, "auto")


def _divisors(n: int):
    out = set()
    i = 1
    while i * i <= n:
        if n % i == 0:
            out.add(i)
            out.add(n // i)
        i += 1
    return sorted(out, reverse=True)


def _grouping(n_out: int, S: int):
    """Group id and rank of every output row for the positions split S."""
    C = n_out // S
    o = np.arange(n_out, dtype=np.int64)
    c, s = o // S, o % S
    if C <= TILE_M:
        pp = TILE_M // C
        g = s // pp
    else:
        cb = -(-C // TILE_M)
        g = s * cb + c // TILE_M
    return g


def _evaluate(g_row, rowptr, col, n_in, P, cols):
    counts = np.diff(rowptr)
    g_tap = np.repeat(g_row, counts)
    keys = np.unique(g_tap * n_in + col)
    G = int(g_row.max()) + 1 if g_row.size else 0
    kg = np.bincount(keys // n_in, minlength=G)
    chunks = float(np.maximum(1, (kg + CHUNK - 1) // CHUNK).sum())
    ntiles = cols // TILE_N
    t = (n_in * cols * (8 + P) / R_HBM + chunks * ntiles * T_CHUNK * P / 7.0 / N_SM
         + G * ntiles * T_TILE / N_SM)
    return t, keys, kg


def build(mac, n_in: int, P: int, cols: int, force: bool = False, device: str = "cuda"):
    """The tensor-core lowering of a _Mac (None when not eligible or slower)."""
    if mac.host is None or not mac.no_rot or mac.max_abs_coef > 127 or P < 5 or P > 8 or cols % TILE_N:
        return None
    rowptr, col, coef = mac.host
    n_out = mac.n_out
    if n_out == 0 or len(col) == 0:
        return None
    nnz = len(col)
    est_sparse = max(nnz * cols / R_SPARSE, (n_in + n_out) * cols * 8 / R_SPARSE_IO)
    best = None
    for S in _divisors(n_out):
        if n_out // S > 4096:
            continue
        g_row = _grouping(n_out, S)
        t, keys, kg = _evaluate(g_row, rowptr, col, n_in, P, cols)
        if best is None or t < best[0]:
            best = (t, S, g_row, keys, kg)
    est_tc, S, g_row, keys, kg = best
    if not force and est_tc >= 0.9 * est_sparse:
        return None
    G = int(g_row.max()) + 1
    empty = np.nonzero(kg == 0)[0]
    if empty.size:  # a group of empty rows (reference: Ciphertext.zero) still needs one zero-weight chunk
        keys = np.union1d(keys, empty.astype(np.int64) * n_in)
        kg = np.bincount(keys // n_in, minlength=G)
    # rows sorted by group (stable: ascending output index inside a group)
    order = np.argsort(g_row, kind="stable")
    m_count = np.bincount(g_row, minlength=G)
    if m_count.max() > TILE_M:
        return None
    row_off = np.concatenate([[0], np.cumsum(m_count)[:-1]])
    rank = np.empty(n_out, dtype=np.int64)
    rank[order] = np.arange(n_out) - np.repeat(row_off, m_count)
    k_off = np.concatenate([[0], np.cumsum(kg)[:-1]])  # offsets into `keys`
    nch = (kg + CHUNK - 1) // CHUNK
    w_off = np.concatenate([[0], np.cumsum(nch)[:-1]])
    # the device list pads every group to a multiple of 4 entries (the
    # kernel copies indices in 16-byte pieces) and the array by one chunk
    kpad = (kg + 3) // 4 * 4
    k_dev = np.concatenate([[0], np.cumsum(kpad)[:-1]])
    kidx = np.zeros(int(kpad.sum()) + CHUNK, dtype=np.int32)
    pos = np.repeat(k_dev - k_off, kg) + np.arange(int(kg.sum()))
    kidx[pos] = (keys % n_in).astype(np.int32)
    # weights into their tiles
    counts = np.diff(rowptr)
    rows_of_tap = np.repeat(np.arange(n_out, dtype=np.int64), counts)
    g_tap = g_row[rows_of_tap]
    kglob = np.searchsorted(keys, g_tap * n_in + col)
    kpos = kglob - k_off[g_tap]
    m = rank[rows_of_tap]
    tile = w_off[g_tap] + kpos // CHUNK
    kk = kpos % CHUNK
    off = tile * TILE_BYTES + (m // 8) * (CHUNK // 16 * 128) + (kk // 16) * 128 + (m % 8) * 16 + kk % 16
    acc = np.zeros(int(nch.sum()) * TILE_BYTES, dtype=np.int32)
    np.add.at(acc, off, np.asarray(coef, dtype=np.int64).astype(np.int32))
    if np.abs(acc).max() > 127:
        return None
    # int32 sums of K products of a byte and a weight stay exact
    if int(kg.max()) * int(np.abs(acc).max()) * 255 * (1 << 24) * 1.01 >= 2.0 ** 53:
        return None
    grp = np.zeros((G, 8), dtype=np.int32)
    grp[:, 0] = row_off
    grp[:, 1] = m_count
    grp[:, 2] = k_dev
    grp[:, 3] = kg
    grp[:, 4] = w_off
    import torch

    d = device
    return TcPlan(
        torch.as_tensor(grp, device=d),
        torch.as_tensor(kidx, device=d),
        torch.as_tensor(order.astype(np.int32), device=d),
        torch.as_tensor(acc.astype(np.int8), device=d),
        G, n_out, S, est_tc, est_sparse,
    )


def plan_for(params, mac, n_in: int):
    """Cached per (_Mac, planes, columns, inputs); None -> use the sparse kernel."""
    mode = _mode()
    if mode == "off":
        return None
    h = params.native()
    L = _lib.lib()
    P = L.fcn_tc_planes(h.ptr)
    cols = 2 * len(params.limb_primes) * params.n
    key = (P, cols, n_in, mode)
    if key not in mac.tc:
        mac.tc[key] = build(mac, n_in, P, cols, force=(mode == "on"))
    return mac.tc[key]


def decode(tcp: TcPlan):
    """(output row, input index, coefficient) of every nonzero weight of a
    lowering -- the inverse of `build`'s tile layout (test helper)."""
    grp = tcp.groups.cpu().numpy()
    kidx = tcp.kidx.cpu().numpy()
    rows = tcp.rows.cpu().numpy()
    w = tcp.wimg.cpu().numpy().astype(np.int64)
    out = []
    for row_off, m, k_off, n_k, w_off, *_ in grp:
        for c in range((n_k + CHUNK - 1) // CHUNK):
            t = w[(w_off + c) * TILE_BYTES:(w_off + c + 1) * TILE_BYTES].reshape(16, CHUNK // 16, 8, 16)  # [m/8][k/16][m%8][k%16]
            mm, kb, mi, ki = np.nonzero(t)
            mrow = mm * 8 + mi
            kk = c * CHUNK + kb * 16 + ki
            assert np.all(mrow < m) and np.all(kk < n_k)
            out += list(zip(rows[row_off + mrow].tolist(), kidx[k_off + kk].tolist(), t[mm, kb, mi, ki].tolist()))
    return sorted(out)


def run(params, tcp: TcPlan, cur, out, fanout=(), lo: int = 0, hi: int | None = None):
    """Rows [lo, hi) of the layer into `out` (and every fan-out pointer)."""
    import torch

    hi = tcp.n_out if hi is None else hi
    h = params.native()
    L = _lib.lib()
    P = L.fcn_tc_planes(h.ptr)
    n_in = cur.shape[0]
    cols = 2 * len(params.limb_primes) * params.n
    planes = torch.empty(L.fcn_tc_planes_bytes(h.ptr, n_in), dtype=torch.uint8, device=cur.device)
    st = dev.stream_ptr()
    _lib.check(L.fcn_split_planes(h.ptr, cur.data_ptr(), n_in, planes.data_ptr(), st))
    ptrs = _lib.ptr_array([out.data_ptr()] + [int(p) for p in fanout])
    import ctypes as C

    _lib.check(L.fcn_linear_mac_tc(h.ptr, planes.data_ptr(), n_in, tcp.n_groups, tcp.groups.data_ptr(),
                                   tcp.kidx.data_ptr(), tcp.rows.data_ptr(), tcp.wimg.data_ptr(),
                                   C.cast(ptrs, C.c_void_p), 1 + len(fanout), lo, hi, st))
    return out
