// libfcn: batched negacyclic NTT on B200 (replaces reference ring.py:199-255).
//
// Two kernel families produce bit-identical outputs (canonical residues,
// forward output in the reference's bit-reversed order):
//
//  * ntt_v2 (n = 1024 .. 16384, 2^34 <= q < 2^56): one persistent CTA per row slot,
//    n/32 threads each owning 32 residues in registers.  A transform is
//    three register passes -- 5 stages, LOGN-10 stages, 5 stages -- with two
//    shared-memory exchanges (row padded by one word per 32 so every access
//    pattern is conflict-free).  The forward transform loads pass-1 operands
//    straight from HBM (coalesced: thread t holds t + j n/32) and prefetches
//    the next row into registers while the finished row is copied out; the
//    inverse streams the next row into shared memory with cp.async while the
//    last pass computes and stores coalesced from registers.  Butterflies
//    use a Shoup product whose quotient drops the low 32x32 partial product
//    (3 IMAD instead of 5; remainder in [0,4q)) with Harvey lazy ranges
//    [0,8q) forward / [0,4q) inverse, one canonicalisation at the end, and
//    the inverse's n^-1 scaling merged into its last stage.
//
//  * ntt_v1 (any other n, or q >= 2^61): the generic shared-memory kernel
//    with exact Shoup products.

#include <cstdlib>
#include <mutex>

#include "fcn_common.cuh"

// min resident CTAs per SM for the v2 kernels (register budget = 64K / (T * minb))
#ifndef FCN_NTT_MINB
#define FCN_NTT_MINB(LOGN) (16384 / (1 << (LOGN)))
#endif

namespace fcn {

__device__ __forceinline__ int phys(int i) { return i + (i >> 5); }

// ============================================================ v1 (generic)

template <int R>
__device__ __forceinline__ void v1_fwd_pass(uint64_t* sm, int logs, int ls0, int sbase, int part,
                                            const Twiddle* __restrict__ tw, uint64_t q, uint64_t q2, bool last) {
  constexpr int G = 1 << R;
  const int lt = logs - ls0 - R;
  const int tend = 1 << lt;
  const int groups = 1 << (logs - R);
  for (int g = threadIdx.x; g < groups; g += blockDim.x) {
    const int b = g >> lt, o = g & (tend - 1);
    const int base = (b << (lt + R)) + o;
    uint64_t x[G];
#pragma unroll
    for (int j = 0; j < G; ++j) x[j] = sm[phys(base + (j << lt))];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int s = sbase + ls0 + u;
      const int tbase = (1 << s) + (part << (ls0 + u)) + (b << u);
      const int h = G >> (u + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << u); ++blk) {
        const Twiddle w = tw[tbase + blk];
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int j = blk * 2 * h + jj;
          uint64_t X = csub(x[j], q2);
          uint64_t T = shoup_lazy(x[j + h], w.w, w.s, q);
          x[j] = X + T;
          x[j + h] = X - T + q2;
        }
      }
    }
    if (last) {
#pragma unroll
      for (int j = 0; j < G; ++j) x[j] = csub(csub(x[j], q2), q);
    }
#pragma unroll
    for (int j = 0; j < G; ++j) sm[phys(base + (j << lt))] = x[j];
  }
}

template <int R>
__device__ __forceinline__ void v1_inv_pass(uint64_t* sm, int logs, int ls0, int logn, int part,
                                            const Twiddle* __restrict__ tw, const LimbConst& c, bool final_scale,
                                            bool canon) {
  constexpr int G = 1 << R;
  const uint64_t q = c.q, q2 = c.q2;
  const int lt = ls0;
  const int tstart = 1 << lt;
  const int groups = 1 << (logs - R);
  for (int g = threadIdx.x; g < groups; g += blockDim.x) {
    const int b = g >> lt, o = g & (tstart - 1);
    const int base = (b << (lt + R)) + o;
    uint64_t x[G];
#pragma unroll
    for (int j = 0; j < G; ++j) x[j] = sm[phys(base + (j << lt))];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int s = ls0 + u;
      const int hd = 1 << u;
      const bool is_final = final_scale && (s == logn - 1);
      const int tbase = (1 << (logn - s - 1)) + (part << (logs - s - 1)) + (b << (R - 1 - u));
#pragma unroll
      for (int blk = 0; blk < (G >> (u + 1)); ++blk) {
        const Twiddle w = tw[tbase + blk];
#pragma unroll
        for (int jj = 0; jj < hd; ++jj) {
          const int j = blk * 2 * hd + jj;
          uint64_t X = x[j], Y = x[j + hd];
          uint64_t T = X - Y + q2;
          if (is_final) {
            x[j] = shoup(X + Y, c.ninv, c.ninv_s, q);
            x[j + hd] = shoup(T, c.wlast, c.wlast_s, q);
          } else {
            x[j] = csub(X + Y, q2);
            x[j + hd] = shoup_lazy(T, w.w, w.s, q);
          }
        }
      }
    }
    if (canon && !final_scale) {
#pragma unroll
      for (int j = 0; j < G; ++j) x[j] = csub(x[j], q);
    }
#pragma unroll
    for (int j = 0; j < G; ++j) sm[phys(base + (j << lt))] = x[j];
  }
}

__device__ __forceinline__ int v1_pass_count(int logs) {
  int rem = logs - (logs < 5 ? logs : 5);
  return 1 + (rem + 4) / 5;
}
__device__ __forceinline__ int v1_pass_size(int logs, int p, int np) {
  int last = logs < 5 ? logs : 5;
  if (p == np - 1) return last;
  int rem = logs - last, k = np - 1;
  int base = rem / k, extra = rem % k;
  return base + (p < extra ? 1 : 0);
}

template <bool FWD>
__global__ void __launch_bounds__(512) ntt_v1_kernel(uint64_t* __restrict__ data, int64_t n_segs, int logs, int logn,
                                                     int period, int offset, const LimbConst* __restrict__ lcs,
                                                     const Twiddle* __restrict__ tws, const uint64_t* __restrict__ src,
                                                     int src_div) {
  extern __shared__ uint64_t sm[];
  const int S = 1 << logs;
  const int nseg = 1 << (logn - logs);
  const int n = 1 << logn;
  for (int64_t seg = blockIdx.x; seg < n_segs; seg += gridDim.x) {
    const int64_t row = seg >> (logn - logs);
    const int part = (int)(seg & (nseg - 1));
    const int limb = offset + (int)(row % period);
    const LimbConst c = lcs[limb];
    const Twiddle* tw = tws + (int64_t)limb * n;
    uint64_t* p = data + row * (int64_t)n + (int64_t)part * S;
    const uint64_t* ps = src + (row / src_div) * (int64_t)n + (int64_t)part * S;
    for (int i = threadIdx.x; i < S / 2; i += blockDim.x) {
      ulonglong2 v = reinterpret_cast<const ulonglong2*>(ps)[i];
      sm[phys(2 * i)] = v.x;
      sm[phys(2 * i + 1)] = v.y;
    }
    __syncthreads();
    const int np = v1_pass_count(logs);
    int ls = 0;
    if (FWD) {
      for (int pi = 0; pi < np; ++pi) {
        const int R = v1_pass_size(logs, pi, np);
        const bool last = pi == np - 1;
        switch (R) {
          case 1: v1_fwd_pass<1>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
          case 2: v1_fwd_pass<2>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
          case 3: v1_fwd_pass<3>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
          case 4: v1_fwd_pass<4>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
          default: v1_fwd_pass<5>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
        }
        ls += R;
        __syncthreads();
      }
    } else {
      const bool final_scale = logs == logn;
      for (int pi = np - 1; pi >= 0; --pi) {
        const int R = v1_pass_size(logs, pi, np);
        const bool canon = pi == 0;
        switch (R) {
          case 1: v1_inv_pass<1>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
          case 2: v1_inv_pass<2>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
          case 3: v1_inv_pass<3>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
          case 4: v1_inv_pass<4>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
          default: v1_inv_pass<5>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
        }
        ls += R;
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < S / 2; i += blockDim.x) {
      ulonglong2 v;
      v.x = sm[phys(2 * i)];
      v.y = sm[phys(2 * i + 1)];
      reinterpret_cast<ulonglong2*>(p)[i] = v;
    }
    __syncthreads();
  }
}

// forward stage 0 / inverse last stage of n > 16384 rows, in global memory
__global__ void ntt_v1_fwd_stage0(uint64_t* __restrict__ data, int64_t n_rows, int logn, int period, int offset,
                                  const LimbConst* __restrict__ lcs, const Twiddle* __restrict__ tws) {
  const int n = 1 << logn, h = n >> 1;
  const int64_t total = n_rows * h;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / h;
    const int j = (int)(e % h);
    const int limb = offset + (int)(row % period);
    const LimbConst c = lcs[limb];
    const Twiddle w = tws[(int64_t)limb * n + 1];
    uint64_t* p = data + row * n;
    uint64_t X = p[j];
    uint64_t T = shoup_lazy(p[j + h], w.w, w.s, c.q);
    p[j] = X + T;
    p[j + h] = X - T + c.q2;
  }
}

__global__ void ntt_v1_inv_last(uint64_t* __restrict__ data, int64_t n_rows, int logn, int period, int offset,
                                const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn, h = n >> 1;
  const int64_t total = n_rows * h;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / h;
    const int j = (int)(e % h);
    const LimbConst c = lcs[offset + (int)(row % period)];
    uint64_t* p = data + row * n;
    uint64_t X = p[j], Y = p[j + h];
    p[j] = shoup(X + Y, c.ninv, c.ninv_s, c.q);
    p[j + h] = shoup(X - Y + c.q2, c.wlast, c.wlast_s, c.q);
  }
}

// ================================================================= v2

__device__ __forceinline__ Twiddle ld_tw(const Twiddle* p) {
  const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
  return Twiddle{v.x, v.y};
}

// Cooley-Tukey butterfly without reduction: X' = X + wY, Y' = X - wY + 4q.
// Bounds grow by 4q per stage (inputs < q): after <= 14 stages every value
// is < 57q < 2^62 for q < 2^56.
__device__ __forceinline__ void bfly(uint64_t& X, uint64_t& Y, const Twiddle& w, uint64_t nq, uint64_t q4) {
  const uint64_t t = mulw(Y, w.w, w.s, nq);
  const uint64_t x = X;
  X = x + t;
  Y = x + q4 - t;
}

// Forward (natural in, bit-reversed out; reference ring.py:199-217): R
// stages starting at global stage s0 on G = 2^R registers whose elements lie
// in block b of size n/2^s0; pair twiddle psi[2^s + b 2^u + blk].
template <int R>
__device__ __forceinline__ void fwd_ct(uint64_t* x, int s0, int b, const Twiddle* __restrict__ tw, uint64_t nq,
                                       uint64_t q4) {
  constexpr int G = 1 << R;
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int tb = (1 << (s0 + u)) + (b << u);
    const int h = G >> (u + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << u); ++blk) {
      const Twiddle w = ld_tw(tw + tb + blk);
#pragma unroll
      for (int jj = 0; jj < h; ++jj) {
        const int j = blk * 2 * h + jj;
        bfly(x[j], x[j + h], w, nq, q4);
      }
    }
  }
}

// The forward's last five stages for a thread owning 32 contiguous residues
// (group t): twiddles come from the transposed table [u][blk][t] so a warp's
// loads are 32 consecutive 16-byte entries.
__device__ __forceinline__ void fwd_ct_last(uint64_t* x, int t, int T, const Twiddle* __restrict__ tl, uint64_t nq,
                                            uint64_t q4) {
  int off = 0;
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const int h = 32 >> (u + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << u); ++blk) {
      const Twiddle w = ld_tw(tl + off + blk * T + t);
#pragma unroll
      for (int jj = 0; jj < h; ++jj) {
        const int j = blk * 2 * h + jj;
        bfly(x[j], x[j + h], w, nq, q4);
      }
    }
    off += (1 << u) * T;
  }
}

// Inverse as a decimation-in-time transform on the bit-reversed input:
// stage s pairs elements 2^s apart with twiddle ict[2^s + (idx mod 2^s)].
// Registers hold elements base + (j << s0) with base = (block) + o, o < 2^s0.
template <int R>
__device__ __forceinline__ void inv_ct(uint64_t* x, int s0, int o, const Twiddle* __restrict__ tw, uint64_t nq,
                                       uint64_t q4) {
  constexpr int G = 1 << R;
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int hd = 1 << u;
    const int tb = (1 << (s0 + u)) + o;
#pragma unroll
    for (int jj = 0; jj < hd; ++jj) {
      const Twiddle w = ld_tw(tw + tb + (jj << s0));
#pragma unroll
      for (int blk = 0; blk < (G >> (u + 1)); ++blk) {
        const int j = blk * 2 * hd + jj;
        bfly(x[j], x[j + hd], w, nq, q4);
      }
    }
  }
}


template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 32, FCN_NTT_MINB(LOGN))
    ntt_v2_fwd(uint64_t* __restrict__ data, int64_t n_rows, int period, int offset, const LimbConst* __restrict__ lcs,
               const Twiddle* __restrict__ tws, const Twiddle* __restrict__ twl, const uint64_t* __restrict__ src,
               int src_div) {
  constexpr int N = 1 << LOGN, T = N / 32, RM = LOGN - 10, GM = 1 << RM;
  extern __shared__ uint64_t sm[];
  const int tid = threadIdx.x;
  int64_t row = blockIdx.x;
  if (row >= n_rows) return;
  uint64_t x[32];
  {
    const uint64_t* p = src + (row / src_div) * N;
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = p[tid + j * T];
  }
  for (; row < n_rows; row += gridDim.x) {
    const int limb = offset + (int)(row % period);
    const LimbConst& c = lcs[limb];
    const uint64_t q = c.q, nq = c.nq, q4 = 4 * q;
    const uint32_t m32 = c.m32;
    const Twiddle* tw = tws + (int64_t)limb * N;
    // pass 1: stages 0..4 on t + j*T (twiddles uniform across the CTA)
    fwd_ct<5>(x, 0, 0, tw, nq, q4);
#pragma unroll
    for (int j = 0; j < 32; ++j) sm[phys(tid + j * T)] = x[j];
    __syncthreads();
    // pass 2: stages 5 .. 4+RM on groups of GM elements 32 apart
    if (RM > 0) {
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) {
        const int g = tid + i * T;
        const int base = ((g >> 5) << (5 + RM)) + (g & 31);
#pragma unroll
        for (int j = 0; j < GM; ++j) x[i * GM + j] = sm[phys(base + j * 32)];
      }
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) fwd_ct<(RM > 0 ? RM : 1)>(x + i * GM, 5, (tid + i * T) >> 5, tw, nq, q4);
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) {
        const int g = tid + i * T;
        const int base = ((g >> 5) << (5 + RM)) + (g & 31);
#pragma unroll
        for (int j = 0; j < GM; ++j) sm[phys(base + j * 32)] = x[i * GM + j];
      }
      __syncthreads();
    }
    // pass 3: the last 5 stages on 32 contiguous residues, canonical out
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = sm[tid * 33 + j];
    fwd_ct_last(x, tid, T, twl + (int64_t)limb * N, nq, q4);
#pragma unroll
    for (int j = 0; j < 32; ++j) sm[tid * 33 + j] = reduce_small(x[j], m32, q);
    __syncthreads();
    // prefetch the next row's pass-1 operands, then copy this row out (coalesced)
    const int64_t nxt = row + gridDim.x;
    if (nxt < n_rows) {
      const uint64_t* p = src + (nxt / src_div) * N;
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = p[tid + j * T];
    }
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(data + row * N);
#pragma unroll 4
    for (int i = tid; i < N / 2; i += T) {
      ulonglong2 v;
      v.x = sm[phys(2 * i)];
      v.y = sm[phys(2 * i + 1)];
      o2[i] = v;
    }
    __syncthreads();
  }
}

template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 32, FCN_NTT_MINB(LOGN))
    ntt_v2_inv(uint64_t* __restrict__ data, int64_t n_rows, int period, int offset, const LimbConst* __restrict__ lcs,
               const Twiddle* __restrict__ tws, const Twiddle* __restrict__ twists) {
  constexpr int N = 1 << LOGN, T = N / 32, RM = LOGN - 10, GM = 1 << RM;
  extern __shared__ uint64_t sm[];
  const int tid = threadIdx.x;
  int64_t row = blockIdx.x;
  if (row >= n_rows) return;
  {
    const uint64_t* p = data + row * N;
    for (int i = tid; i < N; i += T) cp_async8(&sm[phys(i)], p + i);
    cp_async_commit();
  }
  uint64_t x[32];
  for (; row < n_rows; row += gridDim.x) {
    const int limb = offset + (int)(row % period);
    const LimbConst& c = lcs[limb];
    const uint64_t q = c.q, nq = c.nq, q4 = 4 * q;
    const Twiddle* tw = tws + (int64_t)limb * N;
    const Twiddle* twist = twists + (int64_t)limb * N;
    cp_async_wait_all();
    __syncthreads();
    // pass 1: stages 0..4 on 32 contiguous residues (twiddles uniform)
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = sm[tid * 33 + j];
    inv_ct<5>(x, 0, 0, tw, nq, q4);
#pragma unroll
    for (int j = 0; j < 32; ++j) sm[tid * 33 + j] = x[j];
    __syncthreads();
    // pass 2: stages 5 .. 4+RM on groups of GM elements 32 apart
    if (RM > 0) {
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) {
        const int g = tid + i * T;
        const int base = ((g >> 5) << (5 + RM)) + (g & 31);
#pragma unroll
        for (int j = 0; j < GM; ++j) x[i * GM + j] = sm[phys(base + j * 32)];
      }
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) inv_ct<(RM > 0 ? RM : 1)>(x + i * GM, 5, (tid + i * T) & 31, tw, nq, q4);
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) {
        const int g = tid + i * T;
        const int base = ((g >> 5) << (5 + RM)) + (g & 31);
#pragma unroll
        for (int j = 0; j < GM; ++j) sm[phys(base + j * 32)] = x[i * GM + j];
      }
      __syncthreads();
    }
    // pass 3: last 5 stages on t + j*T; stream the next row in meanwhile
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = sm[phys(tid + j * T)];
    __syncthreads();
    const int64_t nxt = row + gridDim.x;
    if (nxt < n_rows) {
      const uint64_t* p = data + nxt * N;
      for (int i = tid; i < N; i += T) cp_async8(&sm[phys(i)], p + i);
      cp_async_commit();
    }
    inv_ct<5>(x, LOGN - 5, tid, tw, nq, q4);
    // twist by n^-1 psi^-j, canonicalise, store coalesced
    uint64_t* p = data + row * N;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const Twiddle w = ld_tw(twist + tid + j * T);
      uint64_t v = mulw(x[j], w.w, w.s, nq);
      v = csub(v, 2 * q);
      p[tid + j * T] = csub(v, q);
    }
  }
  cp_async_wait_all();
}


// Integer epilogue for the non-FP64 kernels, applied after the transform.
__global__ void ntt_epi_kernel(const uint64_t* __restrict__ data, int64_t n_rows, int logn, int period, int offset,
                               const LimbConst* __restrict__ lcs, const __grid_constant__ NttEpi E) {
  const int64_t total = n_rows << logn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int limb = offset + (int)((e >> logn) % period);
    const LimbConst& c = lcs[limb];
    uint64_t v = data[e];
    if (E.mode == 3) {
      v = addmod(E.add[e], mulmod(v, E.c2[limb], c), c.q);
    } else {
      v = addmod(v, E.add[e], c.q);
      if (E.mode == 2) v = addmod(mulmod(v, E.c2[limb], c), mulmod(E.lin[e], E.c1[limb], c), c.q);
    }
    for (int d = 0; d < E.out.n; ++d) E.out.dst[d][e] = v;
  }
}

// ============================================================== dispatch

static size_t v1_smem(int logs) { return (size_t)((1 << logs) + (1 << logs) / 32 + 2) * sizeof(uint64_t); }
static size_t v2_smem(int logn) { return (size_t)((1 << logn) + (1 << logn) / 32 + 2) * sizeof(uint64_t); }

template <int LOGN, bool FWD>
static const void* v2_ptr() {
  return FWD ? (const void*)ntt_v2_fwd<LOGN> : (const void*)ntt_v2_inv<LOGN>;
}

// Resident CTAs per SM of the integer NTT kernel for 2^logn (per-device setup).
static cudaError_t v2_occupancy(bool fwd, int logn, int* occ) {
  const void* fn = nullptr;
  switch (logn) {
    case 10: fn = fwd ? v2_ptr<10, true>() : v2_ptr<10, false>(); break;
    case 11: fn = fwd ? v2_ptr<11, true>() : v2_ptr<11, false>(); break;
    case 12: fn = fwd ? v2_ptr<12, true>() : v2_ptr<12, false>(); break;
    case 13: fn = fwd ? v2_ptr<13, true>() : v2_ptr<13, false>(); break;
    default: fn = fwd ? v2_ptr<14, true>() : v2_ptr<14, false>(); break;
  }
  return kernel_occupancy(fn, (1 << logn) / 32, v2_smem(logn), occ);
}

static int launch_v1(const fcn_ring* r, uint64_t* d, int64_t n_rows, int period, int offset, bool fwd, cudaStream_t st,
                     const uint64_t* src, int src_div) {
  const int logn = r->logn;
  const int logs = logn < 14 ? logn : 14;
  const int64_t segs = n_rows << (logn - logs);
  int threads = (1 << logs) / 32;
  threads = threads < 32 ? 32 : (threads > 512 ? 512 : threads);
  const size_t smem = v1_smem(logs);
  int64_t grid = segs;
  const int64_t cap = (int64_t)device_sms() * 64;
  {
    int occ = 0;  // per-device dynamic smem attribute
    FCN_CUDA(kernel_occupancy(fwd ? (const void*)ntt_v1_kernel<true> : (const void*)ntt_v1_kernel<false>, threads,
                              smem, &occ));
  }
  if (grid > cap) grid = cap;
  if (fwd) {
    if (logs < logn) {
      if (src != d) {
        // materialise the broadcast source rows, then transform in place
        for (int64_t rr = 0; rr < n_rows; ++rr) {
          cudaError_t e = cudaMemcpyAsync(d + rr * ((int64_t)1 << logn), src + (rr / src_div) * ((int64_t)1 << logn),
                                          sizeof(uint64_t) << logn, cudaMemcpyDeviceToDevice, st);
          if (e != cudaSuccess) return check_cuda(e, "ntt src copy");
        }
        src = d;
        src_div = 1;
      }
      ntt_v1_fwd_stage0<<<grid_for(n_rows << (logn - 1), 256), 256, 0, st>>>(d, n_rows, logn, period, offset, r->d_lc, r->d_fwd);
      FCN_LAUNCH_CHECK("ntt_v1_fwd_stage0");
    }
    ntt_v1_kernel<true><<<(int)grid, threads, smem, st>>>(d, segs, logs, logn, period, offset, r->d_lc, r->d_fwd, src, src_div);
    FCN_LAUNCH_CHECK("ntt_v1_kernel<fwd>");
  } else {
    ntt_v1_kernel<false><<<(int)grid, threads, smem, st>>>(d, segs, logs, logn, period, offset, r->d_lc, r->d_inv, d, 1);
    FCN_LAUNCH_CHECK("ntt_v1_kernel<inv>");
    if (logs < logn) {
      ntt_v1_inv_last<<<grid_for(n_rows << (logn - 1), 256), 256, 0, st>>>(d, n_rows, logn, period, offset, r->d_lc);
      FCN_LAUNCH_CHECK("ntt_v1_inv_last");
    }
  }
  return FCN_OK;
}

template <int LOGN>
static void launch_v2_t(bool fwd, int grid, uint64_t* d, int64_t n_rows, int period, int offset, const fcn_ring* r,
                        cudaStream_t st, const uint64_t* src, int src_div) {
  const size_t sm = v2_smem(LOGN);
  if (fwd)
    ntt_v2_fwd<LOGN><<<grid, (1 << LOGN) / 32, sm, st>>>(d, n_rows, period, offset, r->d_lc, r->d_fwd, r->d_fwd_last,
                                                         src, src_div);
  else
    ntt_v2_inv<LOGN><<<grid, (1 << LOGN) / 32, sm, st>>>(d, n_rows, period, offset, r->d_lc, r->d_ict, r->d_twist);
}

static int launch_epi_int(const fcn_ring* r, const uint64_t* d, int64_t n_rows, int period, int offset, cudaStream_t st,
                          const NttEpi* epi) {
  if (!epi || epi->mode == 0) return FCN_OK;
  ntt_epi_kernel<<<grid_for(n_rows << r->logn, 256), 256, 0, st>>>(d, n_rows, r->logn, period, offset, r->d_lc, *epi);
  FCN_LAUNCH_CHECK("ntt_epi_kernel");
  return FCN_OK;
}

template <int RS>
int launch_ntt_f64(const fcn_ring* r, uint64_t* d, int64_t n_rows, int period, int offset, bool fwd, cudaStream_t st,
                   const uint64_t* src, int src_div, const NttEpi* epi, int sms);  // ntt_f64.cuh

// The FP64 kernels' value bound (ntt_f64.cuh): a butterfly on |Y| <= B q
// adds |t| <= (1/2 + B q 2^-53) q, a reduction leaves |x| <= q/2 + 2^-40 q,
// inputs are canonical (B = 1), and every value must stay below 2^53.
// Returns the cheapest schedule (2, then 1) whose bound holds for limbs up
// to qmax, else 0 (proved for every q < 2^51).  FCN_NTT_RS=0/1/2 caps it.
int f64_schedule(int logn, uint64_t qmax) {
  static const int rs_cap = [] {  // thread-safe one-time read
    const char* ev = getenv("FCN_NTT_RS");
    return (ev && ev[0] >= '0' && ev[0] <= '2') ? ev[0] - '0' : 2;
  }();
  const double e = ((double)qmax + 1.0) * 0x1p-53 * (1.0 + 1e-12);
  for (int rs = rs_cap; rs >= 1; --rs) {
    double B = 1.0;
    bool ok = true;
    for (int s = 0; s < logn && ok; ++s) {
      if (f64_red_before(logn, rs, s)) B = 0.5 + 1e-9;
      B = B + 0.5 + B * e + 1e-9;
      ok = B * e < 1.0;
    }
    if (ok) return rs;
  }
  return 0;
}

}  // namespace fcn

extern "C" int fcn_ntt_f64_schedule(int logn, uint64_t qmax) { return fcn::f64_schedule(logn, qmax); }

namespace fcn {

template <int RS>
int launch_ntt_f64_sq(const fcn_ring* r, const uint64_t* a, const uint64_t* aux, uint64_t* Tout, int64_t units, int k,
                      int m, cudaStream_t st, int sms, bool dbl);  // ntt_f64.cuh

// FCN_NTT_INT=1 selects the integer kernels (A/B tests); read once, thread-safe
static bool force_int() {
  static const bool on = [] {
    const char* ev = getenv("FCN_NTT_INT");
    return ev && ev[0] == '1';
  }();
  return on;
}

int ntt_family(const fcn_ring* r, int period, int offset) {
  const int logn = r->logn;
  bool v2 = logn >= 10 && logn <= 14;
  for (int l = 0; v2 && l < period; ++l) {
    const uint64_t q = r->primes[offset + l];
    v2 = q >= (1ull << 34) && q < (1ull << 56);
  }
  if (!v2) return 0;
  bool f64 = !force_int() && r->d_ffwd;
  for (int l = 0; f64 && l < period; ++l) f64 = r->primes[offset + l] < (1ull << 51);
  return f64 ? 2 : 1;
}

int launch_ntt(const fcn_ring* r, uint64_t* d, int64_t n_rows, int period, int offset, bool fwd, cudaStream_t st,
               const uint64_t* src, int src_div, const NttEpi* epi) {
  if (n_rows <= 0) return FCN_OK;
  if (fwd && epi && !epi->dbl) epi = nullptr;  // a forward takes only the row-format flag
  if (!src) {
    src = d;
    src_div = 1;
  }
  if (!fwd && src != d) return set_error(FCN_ERR_ARG, "out-of-place inverse NTT is not supported");
  const int logn = r->logn;
  const int sms = device_sms();
  const int family = ntt_family(r, period, offset);
  if (epi && epi->ftwist && (family != 2 || epi->mode == 2 || fwd))
    return set_error(FCN_ERR_STATE, "a replacement twist needs an FP64 inverse (epilogue mode 0, 1 or 3)");
  if (epi && epi->dbl && (family != 2 || epi->mode == 2))
    return set_error(FCN_ERR_STATE, "double-format rows need the FP64 kernels");
  if (epi && epi->out_per && (family != 2 || epi->mode == 2 || epi->mode == 0 || fwd || epi->in_per < 1))
    return set_error(FCN_ERR_STATE, "an output row map needs the FP64 epilogue inverse");
  if (family == 0) {
    const int rc = launch_v1(r, d, n_rows, period, offset, fwd, st, src, src_div);
    return rc ? rc : launch_epi_int(r, d, n_rows, period, offset, st, epi);
  }
  const bool f64 = family == 2;
  if (f64 && epi && epi->mode == 2) {  // no fused FP64 form: plain inverse, then the integer epilogue
    const int rc = launch_ntt(r, d, n_rows, period, offset, false, st);
    return rc ? rc : launch_epi_int(r, d, n_rows, period, offset, st, epi);
  }
  if (f64) {
    uint64_t qmax = 0;
    for (int l = 0; l < period; ++l) qmax = r->primes[offset + l] > qmax ? r->primes[offset + l] : qmax;
    switch (f64_schedule(logn, qmax)) {
      case 2: return launch_ntt_f64<2>(r, d, n_rows, period, offset, fwd, st, src, src_div, epi, sms);
      case 1: return launch_ntt_f64<1>(r, d, n_rows, period, offset, fwd, st, src, src_div, epi, sms);
      default: return launch_ntt_f64<0>(r, d, n_rows, period, offset, fwd, st, src, src_div, epi, sms);
    }
  }
  int occ = 1;
  FCN_CUDA(v2_occupancy(fwd, logn, &occ));
  int64_t grid = (int64_t)sms * occ;
  if (grid > n_rows) grid = n_rows;
  switch (logn) {
    case 10: launch_v2_t<10>(fwd, (int)grid, d, n_rows, period, offset, r, st, src, src_div); break;
    case 11: launch_v2_t<11>(fwd, (int)grid, d, n_rows, period, offset, r, st, src, src_div); break;
    case 12: launch_v2_t<12>(fwd, (int)grid, d, n_rows, period, offset, r, st, src, src_div); break;
    case 13: launch_v2_t<13>(fwd, (int)grid, d, n_rows, period, offset, r, st, src, src_div); break;
    default: launch_v2_t<14>(fwd, (int)grid, d, n_rows, period, offset, r, st, src, src_div); break;
  }
  FCN_LAUNCH_CHECK(fwd ? "ntt_v2_fwd" : "ntt_v2_inv");
  return launch_epi_int(r, d, n_rows, period, offset, st, epi);
}

template <int RS>
int launch_ntt_f64_pair(const fcn_ring* r, uint64_t* d, int64_t units, bool scale, cudaStream_t st, const PairEpi* epi,
                        int sms);  // ntt_f64.cuh

int launch_ntt_pair(const fcn_ring* r, uint64_t* d, int64_t units, bool scale, cudaStream_t st, const PairEpi* epi) {
  if (units <= 0) return FCN_OK;
  if (!epi || epi->kq < 3 || epi->kq > kPairLimbs || r->L < epi->kq)
    return set_error(FCN_ERR_ARG, "pair inverse: bad epilogue");
  if (ntt_family(r, epi->kq, 0) != 2) return set_error(FCN_ERR_STATE, "pair inverse needs the FP64 kernels");
  const uint64_t qmax = r->primes[0] > r->primes[1] ? r->primes[0] : r->primes[1];
  const int sms = device_sms();
  switch (f64_schedule(r->logn, qmax)) {
    case 2: return launch_ntt_f64_pair<2>(r, d, units, scale, st, epi, sms);
    case 1: return launch_ntt_f64_pair<1>(r, d, units, scale, st, epi, sms);
    default: return launch_ntt_f64_pair<0>(r, d, units, scale, st, epi, sms);
  }
}

int launch_ntt_square_tensor(const fcn_ring* r, const uint64_t* a, const uint64_t* aux, uint64_t* Tout, int64_t C,
                             int k, int m, cudaStream_t st, bool dbl) {
  if (C <= 0) return FCN_OK;
  if (!r->d_ffwd || r->logn < 10 || r->logn > 14 || r->L != k + m) return 1;
  uint64_t qmax = 0;
  for (int l = 0; l < r->L; ++l) {
    if (r->primes[l] >= (1ull << 51)) return 1;
    qmax = r->primes[l] > qmax ? r->primes[l] : qmax;
  }
  const int sms = device_sms();
  const int64_t units = C * (k + m);
  switch (f64_schedule(r->logn, qmax)) {
    case 2: return launch_ntt_f64_sq<2>(r, a, aux, Tout, units, k, m, st, sms, dbl);
    case 1: return launch_ntt_f64_sq<1>(r, a, aux, Tout, units, k, m, st, sms, dbl);
    default: return launch_ntt_f64_sq<0>(r, a, aux, Tout, units, k, m, st, sms, dbl);
  }
}

}  // namespace fcn
