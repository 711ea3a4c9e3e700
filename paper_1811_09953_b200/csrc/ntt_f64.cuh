// libfcn: FP64-pipe batched negacyclic NTT kernels (replace reference
// ring.py:199-255 for limbs q < 2^51), templated on the transform size and on
// the reduction schedule RS.  Each schedule is instantiated in its own
// translation unit (ntt_f64_s{0,1,2}.cu) so the three compile in parallel.
#pragma once

#include <cstdlib>
#include <mutex>

#include "fcn_common.cuh"

#ifndef FCN_NTT_MINB
#define FCN_NTT_MINB(LOGN) (16384 / (1 << (LOGN)))
#endif

namespace fcn {

__device__ __forceinline__ int phys(int i) { return i + (i >> 5); }
// The forward kernels pad their row buffer by FCN_FWD_PAD words per 32: with
// 2 every thread's 32 contiguous residues start 16-byte aligned, so the
// contiguous phases (pass-3 loads, staging stores, per-warp copy-out) move
// 128 bits per instruction and the copy-out's reads lose their 2-way bank
// conflict (a quarter of the forward's shared-memory wavefronts per row).
#ifndef FCN_FWD_PAD
#define FCN_FWD_PAD 2
#endif
constexpr int kFwdRW = 32 + FCN_FWD_PAD;  // words between consecutive threads' contiguous blocks
__device__ __forceinline__ int physf(int i) { return i + FCN_FWD_PAD * (i >> 5); }
// Experiment (FCN_NTT_STAGGER_NS > 0): the second resident CTA of every SM
// starts this many nanoseconds late, so two CTAs that run identical rows do
// not sit in their memory phases at the same time.
#ifndef FCN_NTT_STAGGER_NS
#define FCN_NTT_STAGGER_NS 0
#endif
// Experiment (-DFCN_NTT_PROF): warp 0 of every CTA of ntt_f64_fwd timestamps
// its phase boundaries (clock64) and adds the deltas into fcn_ntt_prof[]
// (read back with fcn_ntt_prof_read, tools/ntt_phase_prof.py).
#ifdef FCN_NTT_PROF
__device__ unsigned long long fcn_ntt_prof[16];
#define FCN_PROF_DECL unsigned long long pf_t = 0, pf_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define FCN_PROF_ARGS , pf_t, pf_acc
#define FCN_PROF_PARAMS , unsigned long long &pf_t, unsigned long long (&pf_acc)[8]
#define FCN_PROF_START                                            \
  do {                                                            \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(pf_t)::"memory"); \
  } while (0)
#define FCN_PROF_MARK(i)                                          \
  do {                                                            \
    unsigned long long pf_n;                                      \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(pf_n)::"memory"); \
    pf_acc[i] += pf_n - pf_t;                                     \
    pf_t = pf_n;                                                  \
  } while (0)
#define FCN_PROF_FLUSH                                                                \
  do {                                                                                \
    if (threadIdx.x == 0)                                                             \
      for (int pf_i = 0; pf_i < 8; ++pf_i) atomicAdd(&fcn_ntt_prof[pf_i], pf_acc[pf_i]); \
  } while (0)
#else
#define FCN_PROF_DECL
#define FCN_PROF_ARGS
#define FCN_PROF_PARAMS
#define FCN_PROF_START
#define FCN_PROF_MARK(i)
#define FCN_PROF_FLUSH
#endif
__device__ __forceinline__ void stagger_start() {
#if FCN_NTT_STAGGER_NS > 0
  if (blockIdx.x >= (gridDim.x + 1) / 2 && gridDim.x > 148) __nanosleep(FCN_NTT_STAGGER_NS);
#endif
}
// phys(tid + j T) = ps(tid) + j (T + T/32): T is a multiple of 32, so the
// padding of element tid + j T is known at compile time once ps(tid) is
// (the compiler does not derive this itself and spent one LEA per access).
__device__ __forceinline__ int ps_strided(int tid) { return tid + (tid >> 5); }
// pass-2 group i of thread tid: element base + j 32 with g = tid + i T,
// base = ((g >> 5) << (5 + RM)) + (g & 31); phys(base + 32 j) =
// ps_group(tid) + 33 i GM^2 + 33 j.
template <int RM>
__device__ __forceinline__ int ps_group(int tid) {
  return (((tid >> 5) << (5 + RM)) + (tid & 31)) + ((tid >> 5) << RM);
}

// ================================================================= f64
// Same three-pass structure as v2, butterflies on the FP64 pipe with signed
// integer-valued doubles (fcn_common.cuh fmulq/fredq) for limbs q < 2^51.
// Bounds (q < 2^51): for |Y| <= Bq the quotient rint(Y w/q) is within
// 1/2 + B/4 of the exact one (|w| <= q/2, two roundings of 2^-53), so a
// butterfly adds |t| <= (1/2 + B/4) q.  From canonical inputs (B = 1) three
// stages reach B = 3.86; from a reduced |x| <= q/2 + 1, three stages reach
// 2.88.  Every value is therefore reduced before stages 3, 6, 9, 12 and
// nothing ever exceeds 3.86 q < 2^53: all arithmetic is exact (schedule
// RS = 0).  The quotient error is really 1/2 + B q 2^-53, so smaller limbs
// allow fewer reductions: RS = 1 reduces once, before stage LOGN/2, and
// RS = 2 never; launch_ntt (ntt.cu f64_schedule) proves the bound for the
// launch's largest limb before picking either (q just above 2^50: RS = 1,
// one reduction per transform instead of four).

__device__ __forceinline__ double2 ld_ftw(const double2* p) { return __ldg(p); }

__device__ __forceinline__ void fbfly(double& X, double& Y, const double2& w, double q) {
  const double t = fmulq(Y, w.x, w.y, q);
  const double x = X;
  X = x + t;
  Y = x - t;
}

template <int G>
__device__ __forceinline__ void fred_all(double* x, double q, double qi) {
#pragma unroll
  for (int j = 0; j < G; ++j) x[j] = fredq(x[j], qi, q);
}

template <int LOGN, int RS, int R, int S0>
__device__ __forceinline__ void fwd_ctf(double* x, int b, const double2* __restrict__ tw, double q, double qi) {
  constexpr int G = 1 << R;
#pragma unroll
  for (int u = 0; u < R; ++u) {
    if (f64_red_before(LOGN, RS, S0 + u)) fred_all<G>(x, q, qi);
    const int tb = (1 << (S0 + u)) + (b << u);
    const int h = G >> (u + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << u); ++blk) {
      const double2 w = ld_ftw(tw + tb + blk);
#pragma unroll
      for (int jj = 0; jj < h; ++jj) {
        const int j = blk * 2 * h + jj;
        fbfly(x[j], x[j + h], w, q);
      }
    }
  }
}

template <int LOGN, int RS, int S0>
__device__ __forceinline__ void fwd_ctf_last(double* x, int t, int T, const double2* __restrict__ tl, double q,
                                             double qi, double2 w0) {
  int off = 0;
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    if (f64_red_before(LOGN, RS, S0 + u)) fred_all<32>(x, q, qi);
    const int h = 32 >> (u + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << u); ++blk) {
      const double2 w = u == 0 ? w0 : ld_ftw(tl + off + blk * T + t);
#pragma unroll
      for (int jj = 0; jj < h; ++jj) {
        const int j = blk * 2 * h + jj;
        fbfly(x[j], x[j + h], w, q);
      }
    }
    off += (1 << u) * T;
  }
}

template <int LOGN, int RS, int R, int S0, bool PRE = false>
__device__ __forceinline__ void inv_ctf(double* x, int o, const double2* __restrict__ tw, double q, double qi,
                                        double2 w0 = double2{}) {
  constexpr int G = 1 << R;
#pragma unroll
  for (int u = 0; u < R; ++u) {
    if (f64_red_before(LOGN, RS, S0 + u)) fred_all<G>(x, q, qi);
    const int hd = 1 << u;
    const int tb = (1 << (S0 + u)) + o;
#pragma unroll
    for (int jj = 0; jj < hd; ++jj) {
      const double2 w = (PRE && u == 0) ? w0 : ld_ftw(tw + tb + (jj << S0));
#pragma unroll
      for (int blk = 0; blk < (G >> (u + 1)); ++blk) {
        const int j = blk * 2 * hd + jj;
        fbfly(x[j], x[j + hd], w, q);
      }
    }
  }
}

// The forward transform of one row held as signed doubles x[j] = element
// tid + j T: pass 1 (stages 0..4, CTA-uniform twiddles), exchange, pass 2,
// exchange, pass 3 (last five stages; tl = the limb's transposed last-stage
// table).  On return x[j] holds output element 32 tid + j (bit-reversed order),
// not yet reduced.  Starts with a barrier, so the caller may still be reading
// shared memory from the previous row when it calls this.
// The forward keeps phys() addressing in its exchanges: the precomputed
// offsets of the inverse (ps_strided / ps_group) made it 4% slower (measured
// A/B, a different schedule with a small spill).
#define FW_S(j) physf(tid + (j) * T)
#define FW_G(i, j) physf((((tid + (i) * T) >> 5) << (5 + RM)) + ((tid + (i) * T) & 31) + (j) * 32)
template <int LOGN, int RS>
__device__ __forceinline__ void fwd_body(double* x, int tid, double* fs, const double2* __restrict__ tw,
                                         const double2* __restrict__ tl, double q, double qi FCN_PROF_PARAMS) {
  constexpr int N = 1 << LOGN, T = N / 32, RM = LOGN - 10, GM = 1 << RM;
  (void)N;
  // pass 1: stages 0..4 on t + j*T (twiddles uniform across the CTA)
  fwd_ctf<LOGN, RS, 5, 0>(x, 0, tw, q, qi);
  __syncthreads();  // every warp has copied out the previous row
  FCN_PROF_MARK(0);  // load wait + conversions + pass 1 + barrier
#pragma unroll
  for (int j = 0; j < 32; ++j) fs[FW_S(j)] = x[j];
  __syncthreads();
  FCN_PROF_MARK(1);  // exchange 1: stores + barrier
  if (RM > 0) {
#pragma unroll
    for (int i = 0; i < 32 / GM; ++i) {
#pragma unroll
      for (int j = 0; j < GM; ++j) x[i * GM + j] = fs[FW_G(i, j)];
    }
#pragma unroll
    for (int i = 0; i < 32 / GM; ++i) fwd_ctf<LOGN, RS, (RM > 0 ? RM : 1), 5>(x + i * GM, (tid + i * T) >> 5, tw, q, qi);
#pragma unroll
    for (int i = 0; i < 32 / GM; ++i) {
#pragma unroll
      for (int j = 0; j < GM; ++j) fs[FW_G(i, j)] = x[i * GM + j];
    }
  }
  // the first twiddle of pass 3 is requested before the barrier (its L2
  // latency was exposed at the start of the pass)
  const double2 w3 = ld_ftw(tl + tid);
  FCN_PROF_MARK(2);  // pass 2: loads + butterflies + stores
  if (RM > 0) __syncthreads();
  FCN_PROF_MARK(3);  // barrier of exchange 2
  // pass 3: the last 5 stages on 32 contiguous residues
  if (FCN_FWD_PAD == 2) {
    const double2* v2 = reinterpret_cast<const double2*>(fs + tid * kFwdRW);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double2 v = v2[i];
      x[2 * i] = v.x;
      x[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fs[tid * kFwdRW + j];
  }
  fwd_ctf_last<LOGN, RS, LOGN - 5>(x, tid, T, tl, q, qi, w3);
}

// DBL: outputs are the reduced signed residues as raw doubles (|x| <= q/2 +
// 2^-40 q), the internal row format of the square pipeline (no conversion to
// canonical u64 and back between its kernels).
template <int LOGN, int RS, bool DBL = false>
__global__ void __launch_bounds__((1 << LOGN) / 32, FCN_NTT_MINB(LOGN))
    ntt_f64_fwd(uint64_t* __restrict__ data, int64_t n_rows, int period, int offset, const LimbConst* __restrict__ lcs,
                const double2* __restrict__ tws, const double2* __restrict__ twl, const uint64_t* __restrict__ src,
                int src_div) {
  constexpr int N = 1 << LOGN, T = N / 32;
  extern __shared__ uint64_t sm[];
  double* fs = reinterpret_cast<double*>(sm);
  const int tid = threadIdx.x;
  int64_t row = blockIdx.x;
  if (row >= n_rows) return;
  stagger_start();
  double x[32];  // raw u64 bits of the next row between iterations
  {
    const uint64_t* p = src + (src_div == 1 ? row : row / src_div) * N;
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = __longlong_as_double((long long)p[tid + j * T]);
  }
  FCN_PROF_DECL
  FCN_PROF_START;
  for (; row < n_rows; row += gridDim.x) {
    const int limb = offset + (int)(row % period);
    const LimbConst& c = lcs[limb];
    const double q = c.fq, qi = c.fqi;
    const double2* tw = tws + (int64_t)limb * N;
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = u2f((uint64_t)__double_as_longlong(x[j]));
    fwd_body<LOGN, RS>(x, tid, fs, tw, twl + (int64_t)limb * N, q, qi FCN_PROF_ARGS);
    if (FCN_FWD_PAD == 2) {
      ulonglong2* st2 = reinterpret_cast<ulonglong2*>(sm + tid * kFwdRW);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double y0 = fredq(x[2 * i], qi, q), y1 = fredq(x[2 * i + 1], qi, q);
        st2[i] = DBL ? make_ulonglong2((uint64_t)__double_as_longlong(y0), (uint64_t)__double_as_longlong(y1))
                     : make_ulonglong2(f2u_canon(y0, q), f2u_canon(y1, q));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double y = fredq(x[j], qi, q);
        sm[tid * kFwdRW + j] = DBL ? (uint64_t)__double_as_longlong(y) : f2u_canon(y, q);
      }
    }
    FCN_PROF_MARK(4);  // pass 3: loads + butterflies + reduction + staging stores
    // A warp's 32 threads own residues [1024 w, 1024 w + 1024): it copies
    // them out coalesced on its own (no CTA barrier), while the next row's
    // loads are in flight.
    __syncwarp();
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(data + row * N) + (tid & ~31) * 16 + (tid & 31);
    // pair 32 i + lane of this warp's block: thread 2 i + (lane >> 4), residues 2 (lane & 15), + 1
    const uint64_t* sw = sm + ((tid & ~31) + ((tid & 31) >> 4)) * kFwdRW + 2 * (tid & 15);
    const int64_t nxt = row + gridDim.x;
    if (nxt < n_rows) {
      const uint64_t* p = src + (src_div == 1 ? nxt : nxt / src_div) * N;
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = __longlong_as_double((long long)p[tid + j * T]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      ulonglong2 v;
      if (FCN_FWD_PAD == 2) {
        v = *reinterpret_cast<const ulonglong2*>(sw + 2 * kFwdRW * i);
      } else {
        v.x = sw[2 * kFwdRW * i];
        v.y = sw[2 * kFwdRW * i + 1];
      }
      o2[32 * i] = v;
    }
    FCN_PROF_MARK(5);  // next-row loads issued + per-warp copy-out
  }
  FCN_PROF_FLUSH;
}

#ifdef FCN_NTT_PROF
extern "C" int fcn_ntt_prof_read(unsigned long long* out16, int reset);
#endif

// Forward NTT of a squared ciphertext's lifted polys fused with the
// NTT-domain tensor (reference fv.py:511-515 with a = b): a unit (ct, l)
// transforms A0 = NTT(a0 mod b_l) and then A1 = NTT(a1 mod b_l) and writes
// d0 = A0^2, d1 = 2 A0 A1, d2 = A1^2 to Tout[(ct*3 + p)*K + l] (canonical),
// so neither A0 nor A1 makes an HBM round trip through a separate tensor
// kernel.  A0 is parked (centred doubles) in the d2 row by the per-warp
// copy-out and read back by the very thread that wrote it.  Input rows: limb
// l < k from the ciphertexts a ([C][2][k][n]), l >= k from the lift's compact
// auxiliary rows aux ([C][2][m][n]; DBL: signed doubles).  DBL also makes the
// outputs signed doubles.
template <int LOGN, int RS, bool DBL = false>
__global__ void __launch_bounds__((1 << LOGN) / 32, FCN_NTT_MINB(LOGN))
    ntt_f64_fwd_sq(const uint64_t* __restrict__ a, const uint64_t* __restrict__ aux, uint64_t* __restrict__ Tout,
                   int64_t units, int k, int m, const LimbConst* __restrict__ lcs, const double2* __restrict__ tws,
                   const double2* __restrict__ twl) {
  constexpr int N = 1 << LOGN, T = N / 32;
  const int K = k + m;
  extern __shared__ uint64_t sm[];
  double* fs = reinterpret_cast<double*>(sm);
  const int tid = threadIdx.x;
  int64_t u = blockIdx.x;
  if (u >= units) return;
  stagger_start();
  auto src_row = [&](int64_t uu, int ss) -> const uint64_t* {
    const int64_t ct = uu / K;
    const int l = (int)(uu - ct * K);
    return l < k ? a + ((ct * 2 + ss) * k + l) * N : aux + ((ct * 2 + ss) * m + (l - k)) * N;
  };
  double x[32];  // raw u64 bits of the next row between iterations
  {
    const uint64_t* p = src_row(u, 0);
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = __longlong_as_double((long long)p[tid + j * T]);
  }
  const int wb = tid & ~31, ln = tid & 31;
  const int pofs = (wb + (ln >> 4)) * kFwdRW + 2 * (ln & 15);  // this lane's first pair in its warp's block
  int s = 0;
  for (;;) {
    const int64_t ct = u / K;
    const int limb = (int)(u - ct * K);
    const LimbConst& c = lcs[limb];
    const double q = c.fq, qi = c.fqi;
    if (!DBL || limb < k) {  // DBL: the auxiliary rows (limb >= k) arrive as signed doubles from the lift
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = u2f((uint64_t)__double_as_longlong(x[j]));
    }
#ifdef FCN_NTT_PROF
    unsigned long long pf_t = 0, pf_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    fwd_body<LOGN, RS>(x, tid, fs, tws + (int64_t)limb * N, twl + (int64_t)limb * N, q, qi FCN_PROF_ARGS);
    if (FCN_FWD_PAD == 2) {
      double2* st2 = reinterpret_cast<double2*>(fs + tid * kFwdRW);
#pragma unroll
      for (int i = 0; i < 16; ++i) st2[i] = make_double2(fredq(x[2 * i], qi, q), fredq(x[2 * i + 1], qi, q));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) fs[tid * kFwdRW + j] = fredq(x[j], qi, q);  // |.| <= q/2 + 2^-40 q
    }
    __syncwarp();
    const int64_t un = s == 0 ? u : u + gridDim.x;
    const bool more = un < units;
    const uint64_t* pn = more ? src_row(un, s ^ 1) : nullptr;
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(Tout + ((ct * 3 + 2) * K + limb) * N) + wb * 16 + ln;
    const double* fw = fs + pofs;
    if (s == 0) {
      // A0: park it in the d2 row (this warp's block, coalesced) while the A1 row loads
      if (more) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = __longlong_as_double((long long)pn[tid + j * T]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        ulonglong2 v;
        if (FCN_FWD_PAD == 2) {
          v = *reinterpret_cast<const ulonglong2*>(fw + 2 * kFwdRW * i);
        } else {
          v.x = (uint64_t)__double_as_longlong(fw[2 * kFwdRW * i]);
          v.y = (uint64_t)__double_as_longlong(fw[2 * kFwdRW * i + 1]);
        }
        o2[32 * i] = v;
      }
    } else {
      // A1 in shared memory; this lane's parked A0 pairs come back from L2
      // into x[] (free now), each pair replaced by the next row's elements
      // once consumed
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const ulonglong2 v = o2[32 * i];
        x[2 * i] = __longlong_as_double((long long)v.x);
        x[2 * i + 1] = __longlong_as_double((long long)v.y);
      }
      ulonglong2* o0 = reinterpret_cast<ulonglong2*>(Tout + ((ct * 3 + 0) * K + limb) * N) + wb * 16 + ln;
      ulonglong2* o1 = reinterpret_cast<ulonglong2*>(Tout + ((ct * 3 + 1) * K + limb) * N) + wb * 16 + ln;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint64_t t0[2], t1[2], t2[2];
        double2 a1;  // this lane's pair of A1
        if (FCN_FWD_PAD == 2) {
          a1 = *reinterpret_cast<const double2*>(fw + 2 * kFwdRW * i);
        } else {
          a1.x = fw[2 * kFwdRW * i];
          a1.y = fw[2 * kFwdRW * i + 1];
        }
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const double x0 = x[2 * i + v], x1 = v ? a1.y : a1.x;
          const double p0 = fprod(x0, x0, q, qi), mm = fprod(x0, x1, q, qi), p2 = fprod(x1, x1, q, qi);
          const double p1 = fredq(mm + mm, qi, q);
          // DBL: signed doubles, |.| < 0.6 q (the INTT's input bound assumes <= q)
          t0[v] = DBL ? (uint64_t)__double_as_longlong(p0) : f2u_canon(p0, q);
          t1[v] = DBL ? (uint64_t)__double_as_longlong(p1) : f2u_canon(p1, q);
          t2[v] = DBL ? (uint64_t)__double_as_longlong(p2) : f2u_canon(p2, q);
        }
        o0[32 * i] = make_ulonglong2(t0[0], t0[1]);
        o1[32 * i] = make_ulonglong2(t1[0], t1[1]);
        o2[32 * i] = make_ulonglong2(t2[0], t2[1]);
        if (more) {
          x[2 * i] = __longlong_as_double((long long)pn[tid + 2 * i * T]);
          x[2 * i + 1] = __longlong_as_double((long long)pn[tid + (2 * i + 1) * T]);
        }
      }
    }
    if (!more) break;
    u = un;
    s ^= 1;
  }
}

// DBL: rows in and out are signed residues as raw doubles (in: |x| <= q,
// out: |x| <= q/2 + 2^-40 q).
template <int LOGN, int RS, bool DBL = false>
__global__ void __launch_bounds__((1 << LOGN) / 32, FCN_NTT_MINB(LOGN))
    ntt_f64_inv(uint64_t* __restrict__ data, int64_t n_rows, int period, int offset, const LimbConst* __restrict__ lcs,
                const double2* __restrict__ tws, const double2* __restrict__ twists) {
  constexpr int N = 1 << LOGN, T = N / 32, RM = LOGN - 10, GM = 1 << RM;
  extern __shared__ uint64_t sm[];
  double* fs = reinterpret_cast<double*>(sm);
  const int tid = threadIdx.x;
  const int pst = ps_strided(tid), pgr = ps_group<(RM > 0 ? RM : 0)>(tid);
  int64_t row = blockIdx.x;
  if (row >= n_rows) return;
  stagger_start();
  {
    const uint64_t* p = data + row * N;
    {
#pragma unroll
        for (int j = 0; j < 32; ++j) cp_async8(&sm[pst + j * (T + T / 32)], p + tid + j * T);
      }
    cp_async_commit();
  }
  double x[32];
  FCN_PROF_DECL
  FCN_PROF_START;
  for (; row < n_rows; row += gridDim.x) {
    const int limb = offset + (int)(row % period);
    const LimbConst& c = lcs[limb];
    const double q = c.fq, qi = c.fqi;
    const double2* tw = tws + (int64_t)limb * N;
    const double2* twist = twists + (int64_t)limb * N;
    cp_async_wait_all();
    __syncthreads();
    FCN_PROF_MARK(0);  // wait for the streamed row + barrier
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = DBL ? __longlong_as_double((long long)sm[tid * 33 + j]) : u2f(sm[tid * 33 + j]);
    inv_ctf<LOGN, RS, 5, 0>(x, 0, tw, q, qi);
#pragma unroll
    for (int j = 0; j < 32; ++j) fs[tid * 33 + j] = x[j];
    __syncthreads();
    FCN_PROF_MARK(1);  // loads + pass 1 + stores + barrier
    if (RM > 0) {
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) {
#pragma unroll
        for (int j = 0; j < GM; ++j) x[i * GM + j] = fs[pgr + 33 * (i * GM * GM + j)];
      }
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) inv_ctf<LOGN, RS, (RM > 0 ? RM : 1), 5>(x + i * GM, (tid + i * T) & 31, tw, q, qi);
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) {
#pragma unroll
        for (int j = 0; j < GM; ++j) fs[pgr + 33 * (i * GM * GM + j)] = x[i * GM + j];
      }
    }
    const double2 w3 = ld_ftw(tw + (1 << (LOGN - 5)) + tid);  // pass 3's first twiddle, before the barrier
    FCN_PROF_MARK(2);  // pass 2
    if (RM > 0) __syncthreads();
    FCN_PROF_MARK(3);  // barrier of exchange 2
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fs[pst + j * (T + T / 32)];
    // the next row lands in exactly the slots this thread just read: no barrier
    const int64_t nxt = row + gridDim.x;
    if (nxt < n_rows) {
      const uint64_t* p = data + nxt * N;
      {
#pragma unroll
        for (int j = 0; j < 32; ++j) cp_async8(&sm[pst + j * (T + T / 32)], p + tid + j * T);
      }
      cp_async_commit();
    }
    inv_ctf<LOGN, RS, 5, LOGN - 5, true>(x, tid, tw, q, qi, w3);
    FCN_PROF_MARK(4);  // strided loads + next-row copies issued + pass 3 (as scheduled)
    // twist by n^-1 psi^-j, canonicalise, store coalesced
    uint64_t* p = data + row * N;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double2 w = ld_ftw(twist + tid + j * T);
      const double y = fredq(fmulq(x[j], w.x, w.y, q), qi, q);
      p[tid + j * T] = DBL ? (uint64_t)__double_as_longlong(y) : f2u_canon(y, q);
    }
    FCN_PROF_MARK(5);  // twist + reduction + stores
  }
  cp_async_wait_all();
  FCN_PROF_FLUSH;
}

// Inverse with a fused epilogue out = add + v (SCALE: add + c2 v), out of
// place.  The epilogue row `add` streams into shared memory with cp.async
// during the last pass (each thread fetches exactly the residues it will
// combine, so no barrier is needed); the next input row is prefetched into
// registers instead (coalesced, as in the forward kernel).
// DBL: the input rows (data) and the add rows are signed residues as raw
// doubles (|x| <= q), the square pipeline's internal format.
template <int LOGN, int RS, bool SCALE, bool FAN, bool DBL = false>
__global__ void __launch_bounds__((1 << LOGN) / 32, FCN_NTT_MINB(LOGN))
    ntt_f64_inv_epi(const uint64_t* __restrict__ data, int64_t n_rows, int period, int offset,
                    const LimbConst* __restrict__ lcs, const double2* __restrict__ tws,
                    const double2* __restrict__ twists, const __grid_constant__ NttEpi E) {
  constexpr int N = 1 << LOGN, T = N / 32, RM = LOGN - 10, GM = 1 << RM;
  extern __shared__ uint64_t sm[];
  double* fs = reinterpret_cast<double*>(sm);
  const int tid = threadIdx.x;
  const int pst = ps_strided(tid), pgr = ps_group<(RM > 0 ? RM : 0)>(tid);
  int64_t row = blockIdx.x;
  if (row >= n_rows) return;
  stagger_start();
  double x[32];  // raw u64 bits of the next row between iterations
  {
    const uint64_t* p = data + row * N;
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = __longlong_as_double((long long)p[tid + j * T]);
  }
  for (; row < n_rows; row += gridDim.x) {
    const int limb = offset + (int)(row % period);
    const LimbConst& c = lcs[limb];
    const double q = c.fq, qi = c.fqi;
    const double2* tw = tws + (int64_t)limb * N;
    const double2* twist = twists + (int64_t)limb * N;
    // the add / out row of this input row (shared-pair relinearisation: limbs 0, 1 of every poly)
    const int64_t orow = E.out_per ? (row / E.in_per) * E.out_per + row % E.in_per : row;
#pragma unroll
    for (int j = 0; j < 32; ++j) sm[pst + j * (T + T / 32)] = (uint64_t)__double_as_longlong(x[j]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = DBL ? __longlong_as_double((long long)sm[tid * 33 + j]) : u2f(sm[tid * 33 + j]);
    inv_ctf<LOGN, RS, 5, 0>(x, 0, tw, q, qi);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) fs[tid * 33 + j] = x[j];
    __syncthreads();
    if (RM > 0) {
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) {
#pragma unroll
        for (int j = 0; j < GM; ++j) x[i * GM + j] = fs[pgr + 33 * (i * GM * GM + j)];
      }
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) inv_ctf<LOGN, RS, (RM > 0 ? RM : 1), 5>(x + i * GM, (tid + i * T) & 31, tw, q, qi);
#pragma unroll
      for (int i = 0; i < 32 / GM; ++i) {
#pragma unroll
        for (int j = 0; j < GM; ++j) fs[pgr + 33 * (i * GM * GM + j)] = x[i * GM + j];
      }
    }
    const double2 w3 = ld_ftw(tw + (1 << (LOGN - 5)) + tid);  // pass 3's first twiddle, before the barrier
    if (RM > 0) __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fs[pst + j * (T + T / 32)];
    {
      // own slots only: no barrier between these reads and the cp.async writes
      const uint64_t* pa = E.add + orow * N;
#pragma unroll
      for (int j = 0; j < 32; ++j) cp_async8(&sm[pst + j * (T + T / 32)], pa + tid + j * T);
      cp_async_commit();
    }
    inv_ctf<LOGN, RS, 5, LOGN - 5, true>(x, tid, tw, q, qi, w3);
    cp_async_wait_all();
    const double c2 = E.fc2[limb], c2q = E.fc2q[limb];
    uint64_t* po = E.out.dst[0] + orow * N;
    const int nd = E.out.n;
    // the next row's element j is requested as soon as x[j] is consumed, so
    // its loads overlap the rest of this epilogue
    const int64_t nxt = row + gridDim.x;
    const uint64_t* pn = data + (nxt < n_rows ? nxt : row) * N;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double2 w = ld_ftw(twist + tid + j * T);
      double y = fmulq(x[j], w.x, w.y, q);  // |y| < 1.5 q (|x| < 7.5 q)
      if (SCALE) y = fmulq(y, c2, c2q, q);  // |y| < 0.7 q
      const uint64_t ar = sm[pst + j * (T + T / 32)];  // DBL: the add row (R0/R1) is signed doubles too
      const uint64_t v = f2u_canon(fredq(y + (DBL ? __longlong_as_double((long long)ar) : u2f(ar)), qi, q), q);
      po[tid + j * T] = v;
      if (FAN) {  // fan-out to the peers' buffers
        for (int d = 1; d < nd; ++d) E.out.dst[d][orow * N + tid + j * T] = v;
      }
      x[j] = __longlong_as_double((long long)pn[tid + j * T]);
    }
  }
}

// Shared-pair relinearisation (fcn_common.cuh PairEpi): unit u = ((ct, poly),
// j - 2) owns the rows 2u (V_j mod q_0) and 2u + 1 (V_j mod q_1) of `data`
// (signed doubles from the key MAC).  The CTA inverts row 0, parks its
// twisted, reduced residues y0 in place (coalesced; read back from L2 by the
// thread that wrote them), inverts row 1 and combines, per coefficient,
//   u = (y1 - y0) q_0^-1 mod q_1 (centred),  V = y0 + q_0 u  (|V| < q_0 q_1 / 2),
//   out = add + c2 (y0 + [q_0]_{q_j} u)  (mod q_j, canonical)
// with the add row (R0 / R1) streamed into the thread's own shared-memory
// slots during the last pass, as in ntt_f64_inv_epi.
template <int LOGN, int RS, bool SCALE, bool FAN>
__global__ void __launch_bounds__((1 << LOGN) / 32, FCN_NTT_MINB(LOGN))
    ntt_f64_inv_pair(uint64_t* __restrict__ data, int64_t units, const LimbConst* __restrict__ lcs,
                     const double2* __restrict__ tws, const double2* __restrict__ twists,
                     const __grid_constant__ PairEpi E) {
  constexpr int N = 1 << LOGN, T = N / 32, RM = LOGN - 10, GM = 1 << RM;
  extern __shared__ uint64_t sm[];
  double* fs = reinterpret_cast<double*>(sm);
  const int tid = threadIdx.x;
  const int pst = ps_strided(tid), pgr = ps_group<(RM > 0 ? RM : 0)>(tid);
  int64_t u = blockIdx.x;
  if (u >= units) return;
  stagger_start();
  // every input row streams into the thread's own strided slots with
  // cp.async (as in ntt_f64_inv): row 1 while row 0's last pass runs, the next
  // unit's row 0 slot by slot as the combine consumes the add row
  {
    const uint64_t* p = data + 2 * u * N;
#pragma unroll
    for (int j = 0; j < 32; ++j) cp_async8(&sm[pst + j * (T + T / 32)], p + tid + j * T);
    cp_async_commit();
  }
  double x[32];
  const int kp = E.kq - 2;
  for (; u < units; u += gridDim.x) {
    const int64_t grp = u / kp;
    const int lj = 2 + (int)(u - grp * kp);
    const int64_t orow = grp * E.kq + lj;
    double* row0 = reinterpret_cast<double*>(data + 2 * u * N);
#pragma unroll 1
    for (int s = 0; s < 2; ++s) {
      const LimbConst& c = lcs[s];
      const double q = c.fq, qi = c.fqi;
      const double2* tw = tws + (int64_t)s * N;
      const double2* twist = twists + (int64_t)s * N;
      cp_async_wait_all();
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = __longlong_as_double((long long)sm[tid * 33 + j]);
      inv_ctf<LOGN, RS, 5, 0>(x, 0, tw, q, qi);
#pragma unroll
      for (int j = 0; j < 32; ++j) fs[tid * 33 + j] = x[j];
      __syncthreads();
      if (RM > 0) {
#pragma unroll
        for (int i = 0; i < 32 / GM; ++i) {
#pragma unroll
          for (int j = 0; j < GM; ++j) x[i * GM + j] = fs[pgr + 33 * (i * GM * GM + j)];
        }
#pragma unroll
        for (int i = 0; i < 32 / GM; ++i)
          inv_ctf<LOGN, RS, (RM > 0 ? RM : 1), 5>(x + i * GM, (tid + i * T) & 31, tw, q, qi);
#pragma unroll
        for (int i = 0; i < 32 / GM; ++i) {
#pragma unroll
          for (int j = 0; j < GM; ++j) fs[pgr + 33 * (i * GM * GM + j)] = x[i * GM + j];
        }
      }
      const double2 w3 = ld_ftw(tw + (1 << (LOGN - 5)) + tid);
      if (RM > 0) __syncthreads();
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = fs[pst + j * (T + T / 32)];
      {
        // own slots only: no barrier between these reads and the cp.async
        // writes.  s = 0: row 1 of the unit; s = 1: the add row (R0 / R1)
        const uint64_t* pa = s == 0 ? data + (2 * u + 1) * N : E.add + orow * N;
#pragma unroll
        for (int j = 0; j < 32; ++j) cp_async8(&sm[pst + j * (T + T / 32)], pa + tid + j * T);
        cp_async_commit();
      }
      inv_ctf<LOGN, RS, 5, LOGN - 5, true>(x, tid, tw, q, qi, w3);
      if (s == 0) {
        // y0 = V mod q_0, |y0| <= q_0/2 + 2^-40 q_0: parked in place
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const double2 w = ld_ftw(twist + tid + j * T);
          __stcg(row0 + tid + j * T, fredq(fmulq(x[j], w.x, w.y, q), qi, q));
        }
      } else {
        const LimbConst& cj = lcs[lj];
        const double qj = cj.fq, qji = cj.fqi;
        const double c0 = E.c0[lj], c0q = E.c0q[lj];
        const double c2 = E.fc2[lj], c2q = E.fc2q[lj];
        const double i01 = E.inv01, i01q = E.inv01q;
        uint64_t* po = E.out.dst[0] + orow * N;
        const int nd = E.out.n;
        const int64_t nxt = u + gridDim.x;
        const bool more = nxt < units;
        const uint64_t* pn = data + 2 * (more ? nxt : u) * N;
        // parked y0, four coefficients ahead (L2 hits)
        double y0n[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) y0n[j] = __ldcg(row0 + tid + j * T);
        // the twist in a loop of its own: nothing but x[] is live, so the
        // table loads (L2) run several coefficients ahead of their products
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const double2 w = ld_ftw(twist + tid + j * T);
          x[j] = fmulq(x[j], w.x, w.y, q);  // V mod q_1, |y1| < 1.5 q_1
        }
        cp_async_wait_all();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const double y1 = x[j];
          const double y0 = y0n[j & 3];
          if (j + 4 < 32) y0n[j & 3] = __ldcg(row0 + tid + (j + 4) * T);
          // u = (y1 - y0) q_0^-1 mod q_1, |u| <= q_1/2 + 2^-40 q_1 (|y1 - y0| < 1.5 q_1 + 0.51 q_0 < 2^53)
          const double uu = fredq(fmulq(y1 - y0, i01, i01q, q), qi, q);
          // V mod q_j = y0 + [q_0]_{q_j} u: |.| < 1.5 q_j + 0.51 q_0 < 3.6 q_j (limbs within a factor 4)
          double z = fmulq(uu, c0, c0q, qj) + y0;
          if (SCALE) z = fmulq(z, c2, c2q, qj);  // |z| < 1.5 q_j
          const double ar = __longlong_as_double((long long)sm[pst + j * (T + T / 32)]);
          // the slot just read takes the next unit's row 0 (the asm names ar,
          // so the copy cannot be scheduled ahead of the read)
          if (more) cp_async8_after(&sm[pst + j * (T + T / 32)], pn + tid + j * T, ar);
          const uint64_t v = f2u_canon(fredq(z + ar, qji, qj), qj);
          po[tid + j * T] = v;
          if (FAN) {
            for (int d = 1; d < nd; ++d) E.out.dst[d][orow * N + tid + j * T] = v;
          }
        }
        cp_async_commit();
      }
    }
  }
  cp_async_wait_all();
}

// ============================================================== dispatch

// Resident CTAs per SM of one kernel (dynamic smem attribute set per device).
template <int LOGN, int RS, int V>
struct F64Occ {
  static int get(const void* fn, size_t smem, cudaError_t* err) {
    int occ = 1;
    *err = kernel_occupancy(fn, (1 << LOGN) / 32, smem, &occ);
    return occ;
  }
};

// Launch one FP64 NTT kernel with the grid its occupancy allows.
template <int LOGN, int RS, int V, class Kern, class... Args>
static int f64_go(Kern kern, int sms, int64_t n_rows, size_t sm, cudaStream_t st, Args... args) {
  cudaError_t err = cudaSuccess;
  const int occ = F64Occ<LOGN, RS, V>::get((const void*)kern, sm, &err);
  if (err != cudaSuccess) return check_cuda(err, "FP64 NTT attributes");
  int64_t g = (int64_t)sms * occ;
  {
    // experiment: FCN_NTT_GRID_CAP limits the resident CTAs (e.g. 148: one per SM)
    static const int cap = [] {
      const char* ev = getenv("FCN_NTT_GRID_CAP");
      return ev ? atoi(ev) : 0;
    }();
    if (cap > 0 && g > cap) g = cap;
  }
  if (g > n_rows) g = n_rows;
  kern<<<(int)g, (1 << LOGN) / 32, sm, st>>>(args...);
  FCN_LAUNCH_CHECK("ntt_f64");
  return FCN_OK;
}

template <int LOGN, int RS>
static int f64_launch_t(bool fwd, int sms, uint64_t* d, int64_t n_rows, int period, int offset, const fcn_ring* r,
                        cudaStream_t st, const uint64_t* src, int src_div, const NttEpi* epi) {
  const size_t smf = (size_t)((1 << LOGN) + FCN_FWD_PAD * ((1 << LOGN) / 32) + 2) * sizeof(uint64_t);
  const size_t sm = (size_t)((1 << LOGN) + (1 << LOGN) / 32 + 2) * sizeof(uint64_t);
  const bool dbl = epi && epi->dbl;
  if (fwd) {
    if (dbl)
      return f64_go<LOGN, RS, 7>(ntt_f64_fwd<LOGN, RS, true>, sms, n_rows, smf, st, d, n_rows, period, offset, r->d_lc,
                                 r->d_ffwd, r->d_ffl, src, src_div);
    return f64_go<LOGN, RS, 0>(ntt_f64_fwd<LOGN, RS, false>, sms, n_rows, smf, st, d, n_rows, period, offset, r->d_lc,
                               r->d_ffwd, r->d_ffl, src, src_div);
  }
  if (!epi || epi->mode == 0) {
    const double2* twist = epi && epi->ftwist ? epi->ftwist : r->d_ftwist;
    if (dbl)
      return f64_go<LOGN, RS, 8>(ntt_f64_inv<LOGN, RS, true>, sms, n_rows, sm, st, d, n_rows, period, offset, r->d_lc,
                                 r->d_fict, twist);
    return f64_go<LOGN, RS, 1>(ntt_f64_inv<LOGN, RS, false>, sms, n_rows, sm, st, d, n_rows, period, offset, r->d_lc,
                               r->d_fict, twist);
  }
  const bool scale = epi->mode != 1, fan = epi->out.n != 1;
  const double2* etwist = epi->ftwist ? epi->ftwist : r->d_ftwist;  // e.g. the c2-scaled twist (mode 1)
#define FCN_EPI_GO(V, SC, FN, DB)                                                                                  \
  if (scale == SC && fan == FN && dbl == DB)                                                                        \
    return f64_go<LOGN, RS, V>(ntt_f64_inv_epi<LOGN, RS, SC, FN, DB>, sms, n_rows, sm, st, d, n_rows, period, offset, \
                               r->d_lc, r->d_fict, etwist, *epi);
  FCN_EPI_GO(2, false, false, false)
  FCN_EPI_GO(3, true, false, false)
  FCN_EPI_GO(4, false, true, false)
  FCN_EPI_GO(5, true, true, false)
  FCN_EPI_GO(9, false, false, true)
  FCN_EPI_GO(10, true, false, true)
  FCN_EPI_GO(11, false, true, true)
  FCN_EPI_GO(12, true, true, true)
#undef FCN_EPI_GO
  return set_error(FCN_ERR_STATE, "no FP64 inverse-NTT epilogue for mode %d", epi->mode);
}

template <int RS>
int launch_ntt_f64(const fcn_ring* r, uint64_t* d, int64_t n_rows, int period, int offset, bool fwd, cudaStream_t st,
                   const uint64_t* src, int src_div, const NttEpi* epi, int sms) {
  switch (r->logn) {
    case 10: return f64_launch_t<10, RS>(fwd, sms, d, n_rows, period, offset, r, st, src, src_div, epi);
    case 11: return f64_launch_t<11, RS>(fwd, sms, d, n_rows, period, offset, r, st, src, src_div, epi);
    case 12: return f64_launch_t<12, RS>(fwd, sms, d, n_rows, period, offset, r, st, src, src_div, epi);
    case 13: return f64_launch_t<13, RS>(fwd, sms, d, n_rows, period, offset, r, st, src, src_div, epi);
    case 14: return f64_launch_t<14, RS>(fwd, sms, d, n_rows, period, offset, r, st, src, src_div, epi);
    default: return set_error(FCN_ERR_ARG, "FP64 NTT: unsupported log n %d", r->logn);
  }
}

template <int LOGN, int RS>
static int f64_pair_launch_t(int sms, const fcn_ring* r, uint64_t* d, int64_t units, bool scale, cudaStream_t st,
                             const PairEpi* epi) {
  const size_t sm = (size_t)((1 << LOGN) + (1 << LOGN) / 32 + 2) * sizeof(uint64_t);
  const bool fan = epi->out.n != 1;
#define FCN_PAIR_GO(V, SC, FN)                                                                                  \
  if (scale == SC && fan == FN)                                                                                 \
    return f64_go<LOGN, RS, V>(ntt_f64_inv_pair<LOGN, RS, SC, FN>, sms, units, sm, st, d, units, r->d_lc, r->d_fict, \
                               r->d_ftwist, *epi);
  FCN_PAIR_GO(14, false, false)
  FCN_PAIR_GO(15, true, false)
  FCN_PAIR_GO(16, false, true)
  FCN_PAIR_GO(17, true, true)
#undef FCN_PAIR_GO
  return FCN_OK;
}

template <int RS>
int launch_ntt_f64_pair(const fcn_ring* r, uint64_t* d, int64_t units, bool scale, cudaStream_t st, const PairEpi* epi,
                        int sms) {
  switch (r->logn) {
    case 10: return f64_pair_launch_t<10, RS>(sms, r, d, units, scale, st, epi);
    case 11: return f64_pair_launch_t<11, RS>(sms, r, d, units, scale, st, epi);
    case 12: return f64_pair_launch_t<12, RS>(sms, r, d, units, scale, st, epi);
    case 13: return f64_pair_launch_t<13, RS>(sms, r, d, units, scale, st, epi);
    case 14: return f64_pair_launch_t<14, RS>(sms, r, d, units, scale, st, epi);
    default: return set_error(FCN_ERR_ARG, "FP64 NTT: unsupported log n %d", r->logn);
  }
}

template <int LOGN, int RS>
static int f64_sq_launch_t(int sms, const fcn_ring* r, const uint64_t* a, const uint64_t* aux, uint64_t* Tout,
                           int64_t units, int k, int m, cudaStream_t st, bool dbl) {
  const size_t sm = (size_t)((1 << LOGN) + FCN_FWD_PAD * ((1 << LOGN) / 32) + 2) * sizeof(uint64_t);
  if (dbl)
    return f64_go<LOGN, RS, 13>(ntt_f64_fwd_sq<LOGN, RS, true>, sms, units, sm, st, a, aux, Tout, units, k, m, r->d_lc,
                                r->d_ffwd, r->d_ffl);
  return f64_go<LOGN, RS, 6>(ntt_f64_fwd_sq<LOGN, RS, false>, sms, units, sm, st, a, aux, Tout, units, k, m, r->d_lc,
                             r->d_ffwd, r->d_ffl);
}

template <int RS>
int launch_ntt_f64_sq(const fcn_ring* r, const uint64_t* a, const uint64_t* aux, uint64_t* Tout, int64_t units, int k,
                      int m, cudaStream_t st, int sms, bool dbl) {
  switch (r->logn) {
    case 10: return f64_sq_launch_t<10, RS>(sms, r, a, aux, Tout, units, k, m, st, dbl);
    case 11: return f64_sq_launch_t<11, RS>(sms, r, a, aux, Tout, units, k, m, st, dbl);
    case 12: return f64_sq_launch_t<12, RS>(sms, r, a, aux, Tout, units, k, m, st, dbl);
    case 13: return f64_sq_launch_t<13, RS>(sms, r, a, aux, Tout, units, k, m, st, dbl);
    case 14: return f64_sq_launch_t<14, RS>(sms, r, a, aux, Tout, units, k, m, st, dbl);
    default: return set_error(FCN_ERR_ARG, "FP64 NTT: unsupported log n %d", r->logn);
  }
}

}  // namespace fcn
