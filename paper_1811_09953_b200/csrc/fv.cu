// libfcn: FV evaluation on B200 -- context constants, relinearisation keys,
// fused sparse linear layer, exact ciphertext multiplication, decrypt rounding.
//
// Replaces reference fv.py (EncryptionParams :42-124, add_pt :418-431,
// mul_pt :439-460, mul_ct :463-549, decrypt :337-353) and the per-output
// inner loop of engine.eval_encrypted (engine.py:698-772).
//
// Exactness: the reference computes mul_ct with Python
// big integers.  Here every big-integer step is an RNS identity whose only
// approximate ingredient is a float64 estimate of a *small* integer
// (a CRT overflow count or a floor of a sum of fractions < k+1); each such
// estimate is either provably far from a rounding boundary (the extended
// base leaves >= 3 bits of headroom) or checked against an epsilon band and
// recomputed with exact multiword arithmetic when inside it.  Outputs are
// therefore bit-identical to the reference for every input.

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "bigint.hpp"
#include <cstdlib>

#include "fcn_common.cuh"

namespace fcn {


constexpr int KQ_LIM = 16;  // max ciphertext limbs
constexpr int KE_LIM = 32;  // max extended-base limbs
constexpr int MW_LIM = 18;  // multiword scratch words
constexpr int LANE_LIM = 8;
constexpr double kEps = 1.0 / (1ull << 36);  // ambiguity band of float64 floors

// Per-(context, lane) constants for lift / rescale / digits / decrypt.
struct MulCtConst {
  int k, K, m, D, w, qwords, direct, dwords;
  uint64_t t;
  // lift: y_i = x_i (q/q_i)^-1 mod q_i; aux residue = sum y_i [q/q_i]_{p_j} - v' [q]_{p_j}
  uint64_t qinv[KQ_LIM], qinv_s[KQ_LIM];
  double rq[KQ_LIM];
  uint64_t lc[KE_LIM][KQ_LIM], lc_s[KE_LIM][KQ_LIM];
  uint64_t lvq[KE_LIM][KQ_LIM + 2];
  // rescale: y_j = T_j (B/b_j)^-1 mod b_j
  uint64_t binv[KE_LIM], binv_s[KE_LIM];
  double rb[KE_LIM];
  uint64_t beta[KQ_LIM], beta_s[KQ_LIM];                 // tP mod q_j
  uint64_t rc[KQ_LIM][KE_LIM], rc_s[KQ_LIM][KE_LIM];     // [floor(tP/q_j)]_{q_i} | [tP/p_j]_{q_i}
  uint64_t rvt[KQ_LIM][KE_LIM + 2];                      // (-v tP) mod q_i, v = 0..K
  double hq;                                             // ((q-1)/2)/q
  // multiword: q, (q-1)/2, q/q_i
  uint64_t qw[MW_LIM], hw[MW_LIM];
  uint64_t Qw[KQ_LIM][MW_LIM];
  // decrypt: t = tq_i q_i + tr_i
  uint64_t tr[KQ_LIM], tr_s[KQ_LIM], tq[KQ_LIM];
  // digits: [2^(64 m)]_{q_l}
  uint64_t dpw[KQ_LIM][4], dpw_s[KQ_LIM][4];
  // add_pt: Delta = q // t mod q_i
  uint64_t delta[KQ_LIM], delta_s[KQ_LIM];
};

}  // namespace fcn

struct fcn_ctx {
  int device = 0;
  int n = 0, logn = 0, k = 0, m = 0, ell = 0, log2_beta = 0, n_lanes = 0;
  std::vector<uint64_t> primes, aux, lanes;
  fcn_ring* ext = nullptr;
  fcn::MulCtConst* d_mc = nullptr;  // [n_lanes]
  std::vector<fcn::MulCtConst> host_mc;
  unsigned long long* d_fallbacks = nullptr;
  bool fp = false;  // every ext prime < 2^51: FP64-pipe lift / rescale kernels
  // FP64 inverse twist of the tensor INTT with the rescale's first factor
  // folded in: {w, w/b_l}, w = n^-1 psi_l^-j (B/b_l)^-1 mod b_l signed
  double2* d_ftwist_binv = nullptr;
  // final-INTT twists of the q-limbs scaled by an activation's c2 (the
  // epilogue's c2 multiply folded into the twist), built on first use
  std::mutex twist_mu;
  std::map<int64_t, double2*> ftwist_c2;
  // Shared-pair relinearisation (decided at creation, pair_relin_setup): the
  // digits are transformed under q_0 and q_1 only and the key-switching sums
  // of limbs j >= 2 are rebuilt from their two residues (fcn_common.cuh PairEpi)
  bool pair = false;
  double pair_inv01 = 0, pair_inv01q = 0;
  double pair_c0[fcn::kPairLimbs] = {}, pair_c0q[fcn::kPairLimbs] = {};
};

struct fcn_keys {
  int device = 0;
  int D = 0, k = 0, n = 0;
  uint64_t* d_g = nullptr;  // [D][k][n] NTT domain
  uint64_t* d_a = nullptr;
  double2* d_fg = nullptr;  // FP64 path: {signed w, w / q_l} of d_g / d_a
  double2* d_fa = nullptr;
  // shared-pair relinearisation: [D][2k-2][n] key words {signed w, w / q_p} in
  // the NTT domain of q_p, p = v & 1; v = 0, 1: the limb-0 / limb-1 keys
  // themselves; v = 2 + 2 (j - 2) + p: the centred lift of the limb-j key
  // residues reduced modulo q_p
  double2* d_pg = nullptr;
  double2* d_pa = nullptr;
};

namespace fcn {

// ------------------------------------------------------------ multiword

template <int NW>
__device__ __forceinline__ void mw_zero(uint64_t (&a)[NW]) {
#pragma unroll
  for (int i = 0; i < NW; ++i) a[i] = 0;
}

// a += y * src (src: nsrc words, little endian)
template <int NW>
__device__ __forceinline__ void mw_mac(uint64_t (&a)[NW], const uint64_t* __restrict__ src, int nsrc, uint64_t y) {
  uint64_t carry = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    if (i < nsrc) {  // a compile-time bound folds the products away past it
      const uint64_t s = src[i];
      uint64_t lo = s * y, hi = __umul64hi(s, y);
      uint64_t t = a[i] + lo;
      hi += t < lo;
      uint64_t t2 = t + carry;
      hi += t2 < carry;
      a[i] = t2;
      carry = hi;
    } else {
      const uint64_t t = a[i] + carry;
      carry = t < carry;
      a[i] = t;
    }
  }
}

template <int NW>
__device__ __forceinline__ void mw_add(uint64_t (&a)[NW], const uint64_t* __restrict__ b) {
  uint64_t c = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    uint64_t s = a[i] + b[i];
    uint64_t c1 = s < b[i];
    uint64_t s2 = s + c;
    c = c1 + (s2 < c);
    a[i] = s2;
  }
}

template <int NW>
__device__ __forceinline__ void mw_sub(uint64_t (&a)[NW], const uint64_t* __restrict__ b) {
  uint64_t br = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    uint64_t d = a[i] - b[i];
    uint64_t b1 = a[i] < b[i];
    uint64_t d2 = d - br;
    br = b1 + (d < br);
    a[i] = d2;
  }
}

// a -= u * b (u small), two's complement
template <int NW>
__device__ __forceinline__ void mw_submul(uint64_t (&a)[NW], const uint64_t* __restrict__ b, uint64_t u) {
  uint64_t carry = 0, br = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    uint64_t lo = b[i] * u, hi = __umul64hi(b[i], u);
    uint64_t p = lo + carry;
    hi += p < lo;
    carry = hi;
    uint64_t d = a[i] - p;
    uint64_t b1 = a[i] < p;
    uint64_t d2 = d - br;
    br = b1 + (d < br);
    a[i] = d2;
  }
}

template <int NW>
__device__ __forceinline__ bool mw_negative(const uint64_t (&a)[NW]) {
  return (int64_t)a[NW - 1] < 0;
}

// a >= b for non-negative a
template <int NW>
__device__ __forceinline__ bool mw_ge(const uint64_t (&a)[NW], const uint64_t* __restrict__ b) {
  int res = 0;  // 0 equal so far (from the top), 1 greater, -1 less
#pragma unroll
  for (int i = NW - 1; i >= 0; --i) {
    if (res == 0) res = a[i] > b[i] ? 1 : (a[i] < b[i] ? -1 : 0);
  }
  return res >= 0;
}

// a <- a - g q with g adjusted so that a lands in [0, q); returns g.
template <int NW>
__device__ __forceinline__ int64_t mw_reduce_q(uint64_t (&a)[NW], const MulCtConst* __restrict__ cc, int64_t g) {
  if (g > 0) mw_submul<NW>(a, cc->qw, (uint64_t)g);
  while (mw_negative<NW>(a)) {
    mw_add<NW>(a, cc->qw);
    --g;
  }
  while (mw_ge<NW>(a, cc->qw)) {
    mw_sub<NW>(a, cc->qw);
    ++g;
  }
  return g;
}

template <int NW>
__device__ __forceinline__ uint64_t mw_word(const uint64_t (&a)[NW], int idx) {
  uint64_t r = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i)
    if (i == idx) r = a[i];
  return r;
}

// floor(sum_j r_j (q/q_j) + (q-1)/2) / q) exactly (the rare fallback of a
// float64 floor of sum r_j/q_j + ((q-1)/2)/q).
template <int NW>
__device__ __noinline__ int64_t exact_frac_floor(const uint64_t* r, int k, const MulCtConst* __restrict__ cc,
                                                 int64_t g_est) {
  uint64_t a[NW];
  mw_zero<NW>(a);
  for (int j = 0; j < k; ++j) mw_mac<NW>(a, cc->Qw[j], cc->qwords, r[j]);
  mw_add<NW>(a, cc->hw);
  return mw_reduce_q<NW>(a, cc, g_est);
}

__device__ __forceinline__ double cc_hq(const MulCtConst* __restrict__ cc) { return __ldg(&cc->hq); }

// ------------------------------------------------------------ add_pt

__global__ void add_plain_kernel(uint64_t* __restrict__ cts, int64_t n_terms, const int32_t* __restrict__ ct_index,
                                 const int32_t* __restrict__ pos, const int64_t* __restrict__ coef, int k, int logn,
                                 const MulCtConst* __restrict__ cc, const LimbConst* __restrict__ lcs) {
  const int64_t total = n_terms * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t term = e / k;
    const int i = (int)(e % k);
    const LimbConst c = lcs[i];
    const int64_t cf = coef[term];
    const uint64_t mag = cf < 0 ? (uint64_t)(-(cf + 1)) + 1 : (uint64_t)cf;
    uint64_t v = shoup(mag, 1, c.one_s, c.q);
    v = shoup(v, cc->delta[i], cc->delta_s[i], c.q);
    if (cf < 0 && v) v = c.q - v;
    uint64_t* p = cts + ((int64_t)ct_index[term] * 2 * k + i) * ((int64_t)1 << logn) + pos[term];
    *p = addmod(*p, v, c.q);
  }
}

// ------------------------------------------------------- linear MAC layer

// out[o] = sum_e coef_e x^rot_e in[col_e]; grid (chunk, output, row = poly*k + limb)
__global__ void __launch_bounds__(256) mac_kernel(const uint64_t* __restrict__ in0, int64_t n_in0,
                                                  const uint64_t* __restrict__ in1, const int32_t* __restrict__ rowptr,
                                                  const int32_t* __restrict__ col, const int32_t* __restrict__ rot,
                                                  const int64_t* __restrict__ coef, const __grid_constant__ Fanout F,
                                                  int logn, int k, const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn;
  const int o = blockIdx.y;
  const int r = blockIdx.z;
  const int limb = r % k;
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (j0 >= n) return;
  const LimbConst c = lcs[limb];
  const int64_t ct_words = (int64_t)2 * k * n;
  uint64_t ph0 = 0, pl0 = 0, nh0 = 0, nl0 = 0, ph1 = 0, pl1 = 0, nh1 = 0, nl1 = 0;
  const int e0 = rowptr[o], e1 = rowptr[o + 1];
  for (int e = e0; e < e1; ++e) {
    const int cl = __ldg(col + e);
    const int rt = __ldg(rot + e);
    const int64_t cf = __ldg(coef + e);
    const uint64_t* src = (cl < n_in0 ? in0 + (int64_t)cl * ct_words : in1 + (int64_t)(cl - n_in0) * ct_words) + (int64_t)r * n;
    const bool neg = cf < 0;
    const uint64_t mag = neg ? (uint64_t)(-(cf + 1)) + 1 : (uint64_t)cf;
    uint64_t x0, x1;
    bool w0 = false, w1 = false;
    if (rt == 0) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + j0);
      x0 = v.x;
      x1 = v.y;
    } else {
      int s0 = j0 - rt, s1 = j0 + 1 - rt;
      w0 = s0 < 0;
      w1 = s1 < 0;
      s0 += w0 ? n : 0;
      s1 += w1 ? n : 0;
      x0 = src[s0];
      x1 = src[s1];
    }
    uint64_t h0, l0, h1, l1;
    if ((mag & (mag - 1)) == 0) {
      const int sh = __ffsll((long long)mag) - 1;
      l0 = x0 << sh;
      l1 = x1 << sh;
      h0 = sh ? x0 >> (64 - sh) : 0;
      h1 = sh ? x1 >> (64 - sh) : 0;
    } else {
      l0 = x0 * mag;
      h0 = __umul64hi(x0, mag);
      l1 = x1 * mag;
      h1 = __umul64hi(x1, mag);
    }
    // sign = neg xor wrapped; route into the positive or negative accumulator
    const uint64_t m0 = (neg != w0) ? ~0ull : 0ull;
    const uint64_t m1 = (neg != w1) ? ~0ull : 0ull;
    add128(nh0, nl0, h0 & m0, l0 & m0);
    add128(ph0, pl0, h0 & ~m0, l0 & ~m0);
    add128(nh1, nl1, h1 & m1, l1 & m1);
    add128(ph1, pl1, h1 & ~m1, l1 & ~m1);
    if (mag >> 40) {  // wide constants: fold so 128-bit accumulators never overflow
      pl0 = reduce128(ph0, pl0, c); ph0 = 0;
      nl0 = reduce128(nh0, nl0, c); nh0 = 0;
      pl1 = reduce128(ph1, pl1, c); ph1 = 0;
      nl1 = reduce128(nh1, nl1, c); nh1 = 0;
    }
  }
  ulonglong2 res;
  res.x = submod(reduce128(ph0, pl0, c), reduce128(nh0, nl0, c), c.q);
  res.y = submod(reduce128(ph1, pl1, c), reduce128(nh1, nl1, c), c.q);
  for (int d = 0; d < F.n; ++d) *reinterpret_cast<ulonglong2*>(F.dst[d] + (int64_t)o * ct_words + (int64_t)r * n + j0) = res;
}

// acc + x m (mod 2^64) for a 32-bit multiplier
__device__ __forceinline__ uint64_t mac32(uint64_t acc, uint64_t x, uint32_t m) {
  uint64_t r;
  asm("{\n\t.reg .u32 xl, xh, al, ah;\n\t.reg .u64 t;\n\t"
      "mov.b64 {xl, xh}, %1;\n\t"
      "mov.b64 {al, ah}, %2;\n\t"
      "mad.lo.u32 ah, xh, %3, ah;\n\t"
      "mov.b64 t, {al, ah};\n\t"
      "mad.wide.u32 %0, xl, %3, t;\n\t}"
      : "=l"(r)
      : "l"(x), "l"(acc), "r"(m));
  return r;
}

#ifndef MAC_WAVES
#define MAC_WAVES 8
#endif
#ifndef MAC_ROWS
#define MAC_ROWS 2
#endif
// Fast path: all rotations 0 (constant plaintexts) and max|coef| * q small
// enough that `fold` consecutive products fit one 64-bit accumulator.  Each
// term is then acc += x |c| per residue (mac32: IMAD.WIDE.U32 + IMAD + carry),
// accumulators are folded back below 4q every `fold` terms.  A thread owns
// four residues of NR rows of the same limb (rows r, r + k: c0 and c1), so
// the term metadata (column, coefficient, source address: uniform-datapath
// work) is amortised over 4 NR residues.
// SGN (with SMALL): one signed accumulator per residue instead of a
// positive and a negative one (acc -/+= x |c| in two's complement, |acc| <
// 2^60 by the host's fold), reduced as reduce_small(acc + OFF) with OFF =
// q ceil(2^60 / q): half the accumulator registers.
template <bool SMALL, int NR, bool SGN = false>
__global__ void __launch_bounds__(256) mac_fast_kernel(const uint64_t* __restrict__ in0, int64_t n_in0,
                                                       const uint64_t* __restrict__ in1,
                                                       const int32_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ col,
                                                       const int64_t* __restrict__ coef, const __grid_constant__ Fanout F,
                                                       int logn, int k, const LimbConst* __restrict__ lcs, int fold,
                                                       int n_out) {
  constexpr int V = 4 * NR;
  const int n = 1 << logn;
  const int r = blockIdx.z;  // first row; the others are r + k, r + 2k, ...
  const int j0 = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (j0 >= n) return;
  const LimbConst& c = lcs[r % k];
  const uint64_t q = c.q, nq = c.nq, one_s = c.one_s;
  const uint32_t m32 = c.m32;
  const int64_t ct_words = (int64_t)2 * k * n;
  const int64_t rstep = (int64_t)k * n;
  const uint64_t off60 = SGN ? q * ((1ull << 60) / q + 1) : 0;
  // outputs o = blockIdx.y + i * gridDim.y: per-CTA setup amortised over several outputs
  for (int o = blockIdx.x; o < n_out; o += gridDim.x) {
    uint64_t pos[V], neg[SGN ? 1 : V];
#pragma unroll
    for (int v = 0; v < V; ++v) pos[v] = 0;
#pragma unroll
    for (int v = 0; v < (SGN ? 1 : V); ++v) neg[v] = 0;
    const int e0 = rowptr[o], e1 = rowptr[o + 1];
    int cnt = 0;
    for (int e = e0; e < e1; ++e) {
      const int cl = __ldg(col + e);
      const int64_t cf = __ldg(coef + e);
      const uint64_t* src = (cl < n_in0 ? in0 + (int64_t)cl * ct_words : in1 + (int64_t)(cl - n_in0) * ct_words) +
                            (int64_t)r * n + j0;
      ulonglong2 va[NR], vb[NR];
#pragma unroll
      for (int h = 0; h < NR; ++h) {
        va[h] = *reinterpret_cast<const ulonglong2*>(src + h * rstep);
        vb[h] = *reinterpret_cast<const ulonglong2*>(src + h * rstep + 2);
      }
      // |c| < 2^32 on this path (fold >= 2)
      const uint32_t m = (uint32_t)(cf >= 0 ? cf : -cf);
      if (SGN && cf < 0) {
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          pos[4 * h + 0] -= mac32(0, va[h].x, m);
          pos[4 * h + 1] -= mac32(0, va[h].y, m);
          pos[4 * h + 2] -= mac32(0, vb[h].x, m);
          pos[4 * h + 3] -= mac32(0, vb[h].y, m);
        }
      } else if (SGN || cf >= 0) {
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          pos[4 * h + 0] = mac32(pos[4 * h + 0], va[h].x, m);
          pos[4 * h + 1] = mac32(pos[4 * h + 1], va[h].y, m);
          pos[4 * h + 2] = mac32(pos[4 * h + 2], vb[h].x, m);
          pos[4 * h + 3] = mac32(pos[4 * h + 3], vb[h].y, m);
        }
      } else if (!SGN) {
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          neg[4 * h + 0] = mac32(neg[4 * h + 0], va[h].x, m);
          neg[4 * h + 1] = mac32(neg[4 * h + 1], va[h].y, m);
          neg[4 * h + 2] = mac32(neg[4 * h + 2], vb[h].x, m);
          neg[4 * h + 3] = mac32(neg[4 * h + 3], vb[h].y, m);
        }
      }
      if (++cnt == fold) {
        cnt = 0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if (SGN) {
            pos[v] = reduce_small(pos[v] + off60, m32, q);
          } else if (SMALL) {
            pos[v] = reduce_small(pos[v], m32, q);
            neg[SGN ? 0 : v] = reduce_small(neg[SGN ? 0 : v], m32, q);
          } else {
            pos[v] = mulw(pos[v], 1, one_s, nq);
            neg[SGN ? 0 : v] = mulw(neg[SGN ? 0 : v], 1, one_s, nq);
          }
        }
      }
    }
    uint64_t res[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (SGN) {
        res[v] = reduce_small(pos[v] + off60, m32, q);
        continue;
      }
      // SMALL: sums kept below 2^62 (fold), reduced by the high-word quotient
      const uint64_t a = SMALL ? reduce_small(pos[v], m32, q) : csub(csub(mulw(pos[v], 1, one_s, nq), 2 * q), q);
      const uint64_t b = SMALL ? reduce_small(neg[SGN ? 0 : v], m32, q) : csub(csub(mulw(neg[SGN ? 0 : v], 1, one_s, nq), 2 * q), q);
      res[v] = submod(a, b, q);
    }
#pragma unroll
    for (int h = 0; h < NR; ++h) {
      const int64_t off = (int64_t)o * ct_words + (int64_t)r * n + h * rstep + j0;
      for (int d = 0; d < F.n; ++d) {  // d > 0: fan-out to the peers' buffers
        *reinterpret_cast<ulonglong2*>(F.dst[d] + off) = make_ulonglong2(res[4 * h], res[4 * h + 1]);
        *reinterpret_cast<ulonglong2*>(F.dst[d] + off + 2) = make_ulonglong2(res[4 * h + 2], res[4 * h + 3]);
      }
    }
  }
}

// ------------------------------------------------------------- mul_ct

// Kernel-parameter constant blocks (constant bank: uniform operands, no
// global loads in the per-coefficient loops), sized by the limb counts.
template <int KQ, int KA>
struct LiftP {
  int k, m, K;
  uint64_t q[KQ], nq[KQ], qinv[KQ], qinv_s[KQ];
  double rq[KQ];
  uint64_t p[KA], np[KA], p_one_s[KA];
  uint64_t lc[KA][KQ], lc_s[KA][KQ];
  uint64_t nqp[KA], nqp_s[KA];  // p_j - (q mod p_j)
  // FP64 path: signed multipliers {w, w/q}
  double fq[KQ], fqinv[KQ], fqinvq[KQ];
  double fp[KA], fpi[KA], flc[KA][KQ], flcq[KA][KQ], fnqp[KA], fnqpq[KA];
};

template <int KQ, int KE>
struct RescaleP {
  int k, K, D, w, direct, dwords;
  uint64_t q[KE], nq[KE], binv[KE], binv_s[KE];
  double rb[KE];
  uint64_t one_s[KQ], rq_dummy[KQ];
  double rq[KQ];
  uint64_t beta[KQ], beta_s[KQ];
  uint64_t rc[KQ][KE], rc_s[KQ][KE];
  uint64_t ntp[KQ], ntp_s[KQ];  // q_i - (tP mod q_i)
  uint64_t qinv[KQ], qinv_s[KQ];
  uint64_t dpw[KQ][3], dpw_s[KQ][3];
  // FP64 path (every ext prime < 2^51): signed multipliers {w, w/q}
  double fb[KE], fbinv[KE], fbinvq[KE];
  double fbeta[KQ], fbetaq[KQ];
  double fq[KQ], fqi[KQ];
  double frc[KQ][KE], frcq[KQ][KE];
  double fntp[KQ], fntpq[KQ];
  // fused activation (FP64 path): R01 rows become c2 R + c1 lin (mod q_i)
  int act;
  // FP64 path: the inputs are already y_j = T_j (B/b_j)^-1 (folded into the INTT's twist)
  int prescaled;
  // ... and stored as signed doubles (|y_j| <= b_j / 2 + 2^-40 b_j), not canonical u64
  int dbl_in;
  double fc2[KQ], fc2q[KQ], fc1[KQ], fc1q[KQ];
};

// canonical x mod q for any x < 2^64 (approximate-quotient product by 1)
__device__ __forceinline__ uint64_t reduce_any(uint64_t x, uint64_t q, uint64_t one_s, uint64_t nq) {
  const uint64_t r = mulw(x, 1, one_s, nq);
  return csub(csub(r, 2 * q), q);
}

// Centered lift of c0/c1 into the extended base (fv.py:463-470):
// y_i = x_i (q/q_i)^-1 (lazy, < 4 q_i), v' = round(sum y_i/q_i) (float64
// with an exact multiword fallback near the tie), aux residue
// = sum y_i [q/q_i]_p - v' [q]_p.
template <int KQ, int KA, int NW>
__global__ void __launch_bounds__(256) lift_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ ext,
                                                   int64_t npoly, int logn, const __grid_constant__ LiftP<KQ, KA> P,
                                                   const MulCtConst* __restrict__ cc,
                                                   unsigned long long* __restrict__ fallbacks) {
  const int n = 1 << logn;
  const int k = P.k, m = P.m, K = P.K;
  const int64_t total = npoly << logn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t poly = e >> logn;
    const int coef = (int)(e & (n - 1));
    uint64_t y[KQ];
    double f = 0.5;
#pragma unroll
    for (int i = 0; i < KQ; ++i) {
      y[i] = 0;
      if (i < k) {
        const uint64_t x = in[(poly * k + i) * n + coef];
        ext[(poly * K + i) * n + coef] = x;
        y[i] = mulw(x, P.qinv[i], P.qinv_s[i], P.nq[i]);
        f += (double)y[i] * P.rq[i];
      }
    }
    int64_t v = (int64_t)floor(f);
    const double fr = f - (double)v;
    if (fr < kEps || fr > 1.0 - kEps) {
      // exact: canonical x = sum y_i Q_i - u q, then v' = u + (x > (q-1)/2)
      uint64_t a[NW];
      mw_zero<NW>(a);
      for (int i = 0; i < k; ++i) mw_mac<NW>(a, cc->Qw[i], cc->qwords, y[i]);
      const int64_t u = mw_reduce_q<NW>(a, cc, (int64_t)floor(f - 0.5));
      bool gt = false, decided = false;
      for (int i = NW - 1; i >= 0; --i) {
        if (!decided && a[i] != cc->hw[i]) {
          gt = a[i] > cc->hw[i];
          decided = true;
        }
      }
      v = u + (gt ? 1 : 0);
      atomicAdd(fallbacks, 1ull);
    }
#pragma unroll
    for (int j = 0; j < KA; ++j) {
      if (j < m) {
        const uint64_t np = P.np[j];
        uint64_t acc = mulw((uint64_t)v, P.nqp[j], P.nqp_s[j], np);
#pragma unroll
        for (int i = 0; i < KQ; ++i)
          if (i < k) acc += mulw(y[i], P.lc[j][i], P.lc_s[j][i], np);
        ext[(poly * K + k + j) * n + coef] = reduce_any(acc, P.p[j], P.p_one_s[j], np);
      }
    }
  }
}

// Constant-multiplier product of the FP64 lift / rescale.  FCN_LR_FRND=1:
// the quotient is rounded by FRND (XU pipe) instead of the magic-constant
// DFMA + DADD: one FP64-pipe operation fewer per product.  The quotient error
// is then 1/2 + |a w/q| 2^-52 (two roundings) instead of 1/2 + |a w/q| 2^-53,
// which is the bound f64_product_period and the 0.7 q product bounds assume.
#ifndef FCN_LR_FRND
#define FCN_LR_FRND 1
#endif
__device__ __forceinline__ double fmulq_lr(double a, double w, double wq, double q) {
#if FCN_LR_FRND
  return fmulq(a, w, wq, q);
#else
  return fmulq_m(a, w, wq, q);
#endif
}

// FP64-pipe variant of lift_kernel (every ext prime < 2^51): y_i signed
// (|y_i| < 0.75 q_i), v = floor(sum y_i/q_i + 1/2) (centred: invariant under
// y_i -> y_i + q_i together with v -> v + 1), aux residues as in
// rescale_f64_kernel with a reduction before every 4th product.  The K input
// loads of the next coefficient are issued before this one computes.
// Instantiated for exact limb counts (k = KQ, m = KA) only.  RP: products
// between reductions of an auxiliary residue (4 for any prime < 2^51, 12
// when every prime is below 2^50.07: f64_product_period).
template <int KQ, int KA, int NW, int RP = 4>
__global__ void __launch_bounds__(256) lift_f64_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ ext,
                                                       int64_t npoly, int logn, const __grid_constant__ LiftP<KQ, KA> P,
                                                       const MulCtConst* __restrict__ cc,
                                                       unsigned long long* __restrict__ fallbacks, int compact) {
  const int n = 1 << logn;
  constexpr int k = KQ, m = KA, K = KQ + KA;  // exact-size instantiations only
  // compact: only the m auxiliary rows are written, as [poly][m][n] (the
  // q-limb rows of the lift are the input rows themselves); compact == 2:
  // as signed doubles (the square pipeline's double-row format)
  const int64_t total = npoly << logn;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr double M = 6755399441055744.0;
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  uint64_t nx[KQ];
  if (e < total) {
#pragma unroll
    for (int i = 0; i < KQ; ++i) nx[i] = i < k ? in[((e >> logn) * k + i) * n + (e & (n - 1))] : 0;
  }
  for (; e < total; e += stride) {
    const int64_t poly = e >> logn;
    const int coef = (int)(e & (n - 1));
    uint64_t cur[KQ];
#pragma unroll
    for (int i = 0; i < KQ; ++i) cur[i] = nx[i];
    if (e + stride < total) {
      const int64_t e2 = e + stride;
#pragma unroll
      for (int i = 0; i < KQ; ++i)
        if (i < k) nx[i] = in[((e2 >> logn) * k + i) * n + (e2 & (n - 1))];
    }
    double y[KQ];
    double f = 0.5;
#pragma unroll
    for (int i = 0; i < KQ; ++i) {
      y[i] = 0.0;
      if (i < k) {
        if (!compact) ext[(poly * K + i) * n + coef] = cur[i];
        y[i] = fmulq_lr(u2f(cur[i]), P.fqinv[i], P.fqinvq[i], P.fq[i]);
        f = fma(y[i], P.rq[i], f);
      }
    }
    double v = floor(f);
    const double fr = f - v;
    if (fr < kEps || fr > 1.0 - kEps) {
      // exact on the canonical y: x = sum y_i Q_i - u q, then v = u + (x > (q-1)/2)
      uint64_t yc[KQ];
      double fc = 0.0;
#pragma unroll
      for (int i = 0; i < KQ; ++i) {
        yc[i] = 0;
        if (i < k) {
          double t = y[i];
          if (t < 0.0) t += P.fq[i];
          y[i] = t;
          yc[i] = (uint64_t)t;
          fc = fma(t, P.rq[i], fc);
        }
      }
      uint64_t a[NW];
      mw_zero<NW>(a);
      for (int i = 0; i < k; ++i) mw_mac<NW>(a, cc->Qw[i], cc->qwords, yc[i]);
      const int64_t u = mw_reduce_q<NW>(a, cc, (int64_t)floor(fc));
      bool gt = false, decided = false;
      for (int i = NW - 1; i >= 0; --i) {
        if (!decided && a[i] != cc->hw[i]) {
          gt = a[i] > cc->hw[i];
          decided = true;
        }
      }
      v = (double)(u + (gt ? 1 : 0));
      atomicAdd(fallbacks, 1ull);
    }
#pragma unroll
    for (int j = 0; j < KA; ++j) {
      if (j < m) {
        const double pj = P.fp[j], pji = P.fpi[j];
        double acc = fmulq_lr(v, P.fnqp[j], P.fnqpq[j], pj);
#pragma unroll
        for (int i = 0; i < KQ; ++i) {
          if (i % RP == RP - 1) acc = fredq(acc, pji, pj);
          acc += fmulq_lr(y[i], P.flc[j][i], P.flcq[j][i], pj);
        }
        const double rr = fredq(acc, pji, pj);
        ext[(compact ? poly * m + j : poly * K + k + j) * n + coef] =
            compact == 2 ? (uint64_t)__double_as_longlong(rr) : f2u_canon(rr, pj);
      }
    }
  }
  (void)M;
}

// NTT-domain tensor: (a0 b0, a0 b1 + a1 b0, a1 b1) per ext limb (fv.py:511-515).
// Two residues per thread (16-byte loads and stores).
__global__ void tensor_kernel(const uint64_t* __restrict__ A, const uint64_t* __restrict__ B, uint64_t* __restrict__ T,
                              int64_t C, int K, int logn, const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn;
  const int64_t total = (C * K) << (logn - 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rowi = e >> (logn - 1);
    const int coef = (int)(e & ((n >> 1) - 1)) * 2;
    const int64_t ct = rowi / K;
    const int j = (int)(rowi % K);
    const LimbConst c = lcs[j];
    const int64_t i0 = ((ct * 2 + 0) * K + j) * n + coef, i1 = ((ct * 2 + 1) * K + j) * n + coef;
    const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(A + i0), a1 = *reinterpret_cast<const ulonglong2*>(A + i1);
    ulonglong2 t0, t1, t2;
    if (B) {
      const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(B + i0), b1 = *reinterpret_cast<const ulonglong2*>(B + i1);
      t0 = make_ulonglong2(mulmod(a0.x, b0.x, c), mulmod(a0.y, b0.y, c));
      t1 = make_ulonglong2(addmod(mulmod(a0.x, b1.x, c), mulmod(a1.x, b0.x, c), c.q),
                           addmod(mulmod(a0.y, b1.y, c), mulmod(a1.y, b0.y, c), c.q));
      t2 = make_ulonglong2(mulmod(a1.x, b1.x, c), mulmod(a1.y, b1.y, c));
    } else {
      t0 = make_ulonglong2(mulmod(a0.x, a0.x, c), mulmod(a0.y, a0.y, c));
      const uint64_t x = mulmod(a0.x, a1.x, c), y = mulmod(a0.y, a1.y, c);
      t1 = make_ulonglong2(addmod(x, x, c.q), addmod(y, y, c.q));
      t2 = make_ulonglong2(mulmod(a1.x, a1.x, c), mulmod(a1.y, a1.y, c));
    }
    *reinterpret_cast<ulonglong2*>(T + ((ct * 3 + 0) * K + j) * n + coef) = t0;
    *reinterpret_cast<ulonglong2*>(T + ((ct * 3 + 1) * K + j) * n + coef) = t1;
    *reinterpret_cast<ulonglong2*>(T + ((ct * 3 + 2) * K + j) * n + coef) = t2;
  }
}

// Base-beta digits of the canonical R2 (fv.py:524-533) from its residues:
// one row per digit when every digit is already < q_i (P.direct), else
// per-limb rows.
// NARROW (FP64 path: every prime < 2^51, exact limb count k = KQ): q has at
// most NQ = ceil(51 KQ / 64) words and q/q_i at most NS = ceil(51 (KQ-1) / 64),
// so the multiword CRT runs on NQ + 1 words with NS-word multiplicands
// instead of NW-word ones (half the 64-bit products at KQ = 4).
template <int KQ, int KE, int NW, bool NARROW = false>
__device__ __forceinline__ void emit_digits(const uint64_t* out, const RescaleP<KQ, KE>& P,
                                            const MulCtConst* __restrict__ cc, uint64_t* __restrict__ DG, int64_t ct,
                                            int coef, int n) {
  const int k = P.k;
  constexpr int NQ = (51 * KQ + 63) / 64;
  constexpr int NA = (NARROW && NQ + 1 < NW) ? NQ + 1 : NW;
  constexpr int NS = NARROW ? ((51 * (KQ - 1) + 63) / 64 < NA ? (51 * (KQ - 1) + 63) / 64 : NA) : NA;
  uint64_t b[NA];
  mw_zero<NA>(b);
  double fu = 0.0;
#pragma unroll
  for (int i = 0; i < KQ; ++i) {
    if (i < k) {
      const uint64_t z = shoup(out[i], P.qinv[i], P.qinv_s[i], P.q[i]);
      fu += (double)z * P.rq[i];
      mw_mac<NA>(b, cc->Qw[i], NARROW ? NS : cc->qwords, z);
    }
  }
  mw_reduce_q<NA>(b, cc, (int64_t)floor(fu));
  uint64_t a[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) a[i] = i < NA ? b[i] : 0;
  const int D = P.D, w = P.w;
  if (P.direct && w == 32) {
    // beta = 2^32 (the configs): digit d is half d&1 of word d>>1 (compile-time indices)
#pragma unroll
    for (int d = 0; d < 2 * NW; ++d)
      if (d < D) DG[(ct * D + d) * n + coef] = (a[d >> 1] >> (32 * (d & 1))) & 0xFFFFFFFFull;
  } else if (P.direct) {
    // every digit < 2^w <= min q_i: one row per digit, broadcast to the limbs by the NTT
    const uint64_t mask = (w >= 64) ? ~0ull : ((1ull << w) - 1);
    for (int d = 0; d < D; ++d) {
      const int bit = d * w;
      const int wi = bit >> 6, bo = bit & 63;
      uint64_t lo = mw_word<NW>(a, wi) >> bo;
      if (bo) lo |= mw_word<NW>(a, wi + 1) << (64 - bo);
      DG[(ct * D + d) * n + coef] = lo & mask;
    }
  } else {
    for (int d = 0; d < D; ++d) {
      const int bit = d * w;
      uint64_t dw[3];
#pragma unroll
      for (int mword = 0; mword < 3; ++mword) {
        const int b0 = bit + 64 * mword;
        const int wi = b0 >> 6, bo = b0 & 63;
        uint64_t lo = mw_word<NW>(a, wi) >> bo;
        if (bo) lo |= mw_word<NW>(a, wi + 1) << (64 - bo);
        const int rem = w - 64 * mword;
        if (rem <= 0) lo = 0;
        else if (rem < 64) lo &= (1ull << rem) - 1;
        dw[mword] = lo;
      }
#pragma unroll
      for (int l = 0; l < KQ; ++l) {
        if (l < k) {
          const uint64_t ql = P.q[l];
          uint64_t val = csub(shoup_lazy(dw[0], 1, P.one_s[l], ql), ql);
          if (P.dwords > 1) val += csub(shoup_lazy(dw[1], P.dpw[l][1], P.dpw_s[l][1], ql), ql);
          if (P.dwords > 2) val += csub(shoup_lazy(dw[2], P.dpw[l][2], P.dpw_s[l][2], ql), ql);
          val = csub(csub(val, 2 * ql), ql);
          DG[((ct * D + d) * k + l) * n + coef] = val;
        }
      }
    }
  }
}

// FP64-pipe tensor (every ext prime < 2^51).  Inputs are centred
// (|a| <= q/2) so a product's quotient estimate rint(ab/q) is within 0.75
// and the remainder |r| <= 0.75 q canonicalises with one conditional add.
__device__ __forceinline__ double fcentre(uint64_t x, uint64_t qh, double q) {
  const double d = u2f(x);
  return x > qh ? d - q : d;
}

__global__ void tensor_f64_kernel(const uint64_t* __restrict__ A, const uint64_t* __restrict__ B, uint64_t* __restrict__ T,
                                  int64_t C, int K, int logn, const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn;
  const int64_t total = (C * K) << (logn - 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rowi = e >> (logn - 1);
    const int coef = (int)(e & ((n >> 1) - 1)) * 2;
    const int64_t ct = rowi / K;
    const int j = (int)(rowi % K);
    const LimbConst& c = lcs[j];
    const uint64_t qh = c.q >> 1;
    const double q = c.fq, qi = c.fqi;
    const int64_t i0 = ((ct * 2 + 0) * K + j) * n + coef, i1 = ((ct * 2 + 1) * K + j) * n + coef;
    const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(A + i0), a1 = *reinterpret_cast<const ulonglong2*>(A + i1);
    const double x0[2] = {fcentre(a0.x, qh, q), fcentre(a0.y, qh, q)};
    const double x1[2] = {fcentre(a1.x, qh, q), fcentre(a1.y, qh, q)};
    uint64_t t0[2], t1[2], t2[2];
    if (B) {
      const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(B + i0), b1 = *reinterpret_cast<const ulonglong2*>(B + i1);
      const double y0[2] = {fcentre(b0.x, qh, q), fcentre(b0.y, qh, q)};
      const double y1[2] = {fcentre(b1.x, qh, q), fcentre(b1.y, qh, q)};
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        t0[v] = f2u_canon(fprod(x0[v], y0[v], q, qi), q);
        t1[v] = f2u_canon(fredq(fprod(x0[v], y1[v], q, qi) + fprod(x1[v], y0[v], q, qi), qi, q), q);
        t2[v] = f2u_canon(fprod(x1[v], y1[v], q, qi), q);
      }
    } else {
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        t0[v] = f2u_canon(fprod(x0[v], x0[v], q, qi), q);
        const double m = fprod(x0[v], x1[v], q, qi);
        t1[v] = f2u_canon(fredq(m + m, qi, q), q);
        t2[v] = f2u_canon(fprod(x1[v], x1[v], q, qi), q);
      }
    }
    *reinterpret_cast<ulonglong2*>(T + ((ct * 3 + 0) * K + j) * n + coef) = make_ulonglong2(t0[0], t0[1]);
    *reinterpret_cast<ulonglong2*>(T + ((ct * 3 + 1) * K + j) * n + coef) = make_ulonglong2(t1[0], t1[1]);
    *reinterpret_cast<ulonglong2*>(T + ((ct * 3 + 2) * K + j) * n + coef) = make_ulonglong2(t2[0], t2[1]);
  }
}

// Exact rescale R = floor((t T + (q-1)/2) / q) mod q from the ext-base
// residues of T (fv.py:473-490, 517-522); for the third tensor poly the
// base-beta digits of R (fv.py:524-533) are emitted instead: one row per
// digit when every digit is already < q_i (P.direct), else per-limb rows.
template <int KQ, int KE, int NW>
__global__ void __launch_bounds__(256, (KQ <= 4 ? 3 : 2)) rescale_kernel(const uint64_t* __restrict__ T, uint64_t* __restrict__ R01,
                                                      uint64_t* __restrict__ DG, int64_t C, int logn,
                                                      const __grid_constant__ RescaleP<KQ, KE> P,
                                                      const MulCtConst* __restrict__ cc,
                                                      unsigned long long* __restrict__ fallbacks) {
  const int n = 1 << logn;
  const int k = P.k, K = P.K;
  const int64_t total = (C * 3) << logn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cp = e >> logn;
    const int coef = (int)(e & (n - 1));
    const int64_t ct = cp / 3;
    const int p = (int)(cp % 3);
    // 1. y_j = T_j (B/b_j)^-1 mod b_j (lazy, < 4 b_j) and the CRT overflow count
    //    v = round(sum y_j / b_j): |T|/B < 1/8 keeps it far from a half
    uint64_t y[KE];
    double fv = 0.0;
#pragma unroll
    for (int j = 0; j < KE; ++j) {
      y[j] = 0;
      if (j < K) {
        const uint64_t x = T[(cp * K + j) * n + coef];
        y[j] = mulw(x, P.binv[j], P.binv_s[j], P.nq[j]);
        fv += (double)y[j] * P.rb[j];
      }
    }
    const uint64_t v = (uint64_t)rint(fv);
    // 2. q-part: y_j tP/q_j = y_j floor(tP/q_j) + h_j + r_j/q_j (exact divmod)
    uint64_t r[KQ];
    uint64_t sh = 0;
    double G = cc_hq(cc);
#pragma unroll
    for (int j = 0; j < KQ; ++j) {
      r[j] = 0;
      if (j < k) {
        uint64_t h;
        r[j] = shoup_divmod(y[j], P.beta[j], P.beta_s[j], P.q[j], &h);
        sh += h;
        G += (double)r[j] * P.rq[j];
      }
    }
    int64_t g = (int64_t)floor(G);
    const double fr = G - (double)g;
    if (fr < kEps || fr > 1.0 - kEps) {
      g = exact_frac_floor<NW>(r, k, cc, g);
      atomicAdd(fallbacks, 1ull);
    }
    // 3. residues of R mod q_i: lazy sums of < 4 q_i products, one reduction
    uint64_t out[KQ];
#pragma unroll
    for (int i = 0; i < KQ; ++i) {
      out[i] = 0;
      if (i < k) {
        const uint64_t qi = P.q[i], nqi = P.nq[i];
        uint64_t acc = mulw(v, P.ntp[i], P.ntp_s[i], nqi);
#pragma unroll
        for (int j = 0; j < KE; ++j) {
          if (j < K) acc += mulw(y[j], P.rc[i][j], P.rc_s[i][j], nqi);
          if (j == 15) acc = mulw(acc, 1, P.one_s[i], nqi);
        }
        acc = reduce_any(acc, qi, P.one_s[i], nqi) + reduce_any(sh, qi, P.one_s[i], nqi) + (uint64_t)g;
        out[i] = csub(csub(acc, qi), qi);
      }
    }
    if (p < 2) {
#pragma unroll
      for (int i = 0; i < KQ; ++i)
        if (i < k) R01[((ct * 2 + p) * k + i) * n + coef] = out[i];
    } else {
      emit_digits<KQ, KE, NW>(out, P, cc, DG, ct, coef, n);
    }
  }
}

// FP64-pipe variant of rescale_kernel for ext primes < 2^51 (same math,
// signed integer-valued doubles, fcn_common.cuh fmulq/fredq):
//  1. y_j = T_j binv_j (|y_j| < 0.75 b_j), v = rint(sum y_j / b_j);
//  2. y_j beta_j = h_j q_j + r_j with any integer h_j (|r_j| < 0.9 q_j):
//     R is invariant under (h_j, r_j) -> (h_j + 1, r_j - q_j), so only the
//     rare exact fallback canonicalises r;
//     (every quotient |a w/q| < 0.75 2^51: magic-constant rounding is exact)
//  3. R mod q_i = sum_j y_j rc_ij + sum h_j + g - v tP, every product
//     |.| < 0.7 q_i, reduced to |.| <= q_i/2 + 1 before products 3, 7, 11..
//     so all partial sums stay below 3.6 q_i < 2^53.
// Instantiated for exact limb counts (k = KQ, K = KE) only.  RP: products
// between reductions in step 3 (4 as above for any prime < 2^51; 12 when
// every prime is below 2^50.07: partial sums < 0.5 + 12 x 0.6 q < 7.7 q < 2^53,
// f64_product_period).
template <int KQ, int KE, int NW, int RP = 4>
#ifndef FCN_RS_MINB
#define FCN_RS_MINB(KQ) ((KQ) <= 4 ? 3 : 2)
#endif
__global__ void __launch_bounds__(256, FCN_RS_MINB(KQ))
    rescale_f64_kernel(const uint64_t* __restrict__ T_in, uint64_t* __restrict__ R01, uint64_t* __restrict__ DG, int64_t C,
                       int logn, const __grid_constant__ RescaleP<KQ, KE> P, const MulCtConst* __restrict__ cc,
                       unsigned long long* __restrict__ fallbacks, const uint64_t* __restrict__ lin) {
  const int n = 1 << logn;
  constexpr int k = KQ, K = KE;  // exact-size instantiations only
  const int64_t total = (C * 3) << logn;
  constexpr int NSH = (KQ + 3) / 4;  // groups of <= 4 quotients (|h_j| < 0.75 2^51): exact sums
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // thread-private two-stage cp.async ring [stage][j][thread]: the K loads of
  // the next coefficient are in flight while this one computes, without
  // holding registers (coalesced: consecutive threads, consecutive words)
  extern __shared__ uint64_t stage_buf[];
  constexpr int SL = KE + KQ;  // staged words per coefficient: K tensor residues (+ k activation inputs)
  const int tid = threadIdx.x, T = blockDim.x;
  const bool act = P.act != 0;
  // (ciphertext, poly) index pairs stay below 2^31 (C 3 rows): 32-bit
  // division by 3, and one base pointer per staged coefficient
  auto stage = [&](int64_t ee, uint64_t* buf) {
    const int cpp = (int)(ee >> logn);
    const int cf = (int)(ee & (n - 1));
    const uint64_t* src = T_in + ((int64_t)cpp * K << logn) + cf;
#pragma unroll
    for (int j = 0; j < KE; ++j) cp_async8(&buf[j * T + tid], src + ((int64_t)j << logn));
    const int ctt = cpp / 3, pp = cpp - 3 * ctt;
    if (act && pp < 2) {
      const uint64_t* ls = lin + ((int64_t)(ctt * 2 + pp) * k << logn) + cf;
#pragma unroll
      for (int i = 0; i < KQ; ++i) cp_async8(&buf[(KE + i) * T + tid], ls + ((int64_t)i << logn));
    }
  };
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < total) stage(e, stage_buf);
  cp_async_commit();
  int sb = 0;
  for (; e < total; e += stride) {
    const int cp32 = (int)(e >> logn);
    const int coef = (int)(e & (n - 1));
    const int64_t ct = cp32 / 3;
    const int p = cp32 - 3 * (int)ct;
    if (e + stride < total) stage(e + stride, stage_buf + (sb ^ 1) * SL * T);
    cp_async_commit();
    cp_async_wait<1>();
    uint64_t cur[KE];
    const uint64_t* cb = stage_buf + sb * SL * T;
#pragma unroll
    for (int j = 0; j < KE; ++j) cur[j] = cb[j * T + tid];
    sb ^= 1;
    double y[KE];
    double fv = 0.0;
#pragma unroll
    for (int j = 0; j < KE; ++j) {
      y[j] = 0.0;
      if (j < K) {
        const double x = P.dbl_in ? __longlong_as_double((long long)cur[j]) : u2f(cur[j]);
        if (P.dbl_in)
          y[j] = x;
        else if (P.prescaled)
          y[j] = x > 0.5 * P.fb[j] ? x - P.fb[j] : x;  // centred: |y_j| <= b_j / 2
        else
          y[j] = fmulq_m(x, P.fbinv[j], P.fbinvq[j], P.fb[j]);
        fv = fma(y[j], P.rb[j], fv);
      }
    }
    const double v = rint(fv);
    double r[KQ];
    double sh[NSH];
#pragma unroll
    for (int g = 0; g < NSH; ++g) sh[g] = 0.0;
    double G = cc_hq(cc);
#pragma unroll
    for (int j = 0; j < KQ; ++j) {
      r[j] = 0.0;
      if (j < k) {
        const double h = y[j] * P.fbeta[j];
        const double l = fma(y[j], P.fbeta[j], -h);
        const double hq = fma(y[j], P.fbetaq[j], 6755399441055744.0) - 6755399441055744.0;
        r[j] = fma(-hq, P.fq[j], h) + l;
        sh[j / 4] += hq;
        G = fma(r[j], P.rq[j], G);
      }
    }
    int64_t g = (int64_t)floor(G);
    const double fr = G - (double)g;
    if (fr < kEps || fr > 1.0 - kEps) {
      uint64_t rc[KQ];
      int64_t corr = 0;
#pragma unroll
      for (int j = 0; j < KQ; ++j) {
        rc[j] = 0;
        if (j < k) {
          double rr = r[j];
          while (rr < 0.0) { rr += P.fq[j]; ++corr; }
          while (rr >= P.fq[j]) { rr -= P.fq[j]; --corr; }
          rc[j] = (uint64_t)rr;
        }
      }
      // floor(G) of the canonical r' = r + corr_j q_j is floor(G) + corr
      g = exact_frac_floor<NW>(rc, k, cc, g + corr) - corr;
      atomicAdd(fallbacks, 1ull);
    }
    const double gd = (double)g;
    double od[KQ];  // R mod q_i, reduced: |.| <= q_i / 2 + 2^-40 q_i
#pragma unroll
    for (int i = 0; i < KQ; ++i) {
      od[i] = 0.0;
      if (i < k) {
        const double qi = P.fq[i], qii = P.fqi[i];
        double acc = gd + fmulq_lr(v, P.fntp[i], P.fntpq[i], qi);
#pragma unroll
        for (int g2 = 0; g2 < NSH; ++g2) acc += fredq(sh[g2], qii, qi);
        if (NSH > 1) acc = fredq(acc, qii, qi);
#pragma unroll
        for (int j = 0; j < KE; ++j) {
          if (j % RP == RP - 1) acc = fredq(acc, qii, qi);
          acc += fmulq_lr(y[j], P.frc[i][j], P.frcq[i][j], qi);
        }
        od[i] = fredq(acc, qii, qi);
      }
    }
    if (p < 2) {
      // R0 / R1 rows for the final INTT's epilogue; dbl_in: as signed doubles
      // like the other rows of the square pipeline
#pragma unroll
      for (int i = 0; i < KQ; ++i) {
        if (i < k) {
          const double qi = P.fq[i], qii = P.fqi[i];
          double r = od[i];
          if (P.act) {
            const double a = u2f(cb[(KE + i) * T + tid]);
            r = fredq(fmulq(r, P.fc2[i], P.fc2q[i], qi) + fmulq(a, P.fc1[i], P.fc1q[i], qi), qii, qi);
          }
          R01[((ct * 2 + p) * k + i) * n + coef] = P.dbl_in ? (uint64_t)__double_as_longlong(r) : f2u_canon(r, qi);
        }
      }
    } else {
      uint64_t out[KQ];
#pragma unroll
      for (int i = 0; i < KQ; ++i) out[i] = i < k ? f2u_canon(od[i], P.fq[i]) : 0;
      emit_digits<KQ, KE, NW, true>(out, P, cc, DG, ct, coef, n);
    }
  }
}

// Key switching MAC in the NTT domain (fv.py:533-537):
// acc0 = sum_d g_d * D_d, acc1 = sum_d a_d * D_d.  A thread owns one
// residue of one limb and walks a range of ciphertexts, so its 2D key words
// are loaded once; the D digit loads of a ciphertext are issued together.
template <int DMAX>
__global__ void __launch_bounds__(256, 4) keymac_kernel(const uint64_t* __restrict__ DG, const uint64_t* __restrict__ kg,
                                                        const uint64_t* __restrict__ ka, uint64_t* __restrict__ ACC,
                                                        int64_t C, int D, int k, int logn,
                                                        const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn;
  const int64_t lc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // l * n + coef
  if (lc >= (int64_t)k * n) return;
  const int l = (int)(lc >> logn);
  const int coef = (int)(lc & (n - 1));
  const LimbConst c = lcs[l];
  uint64_t gk[DMAX], ak[DMAX];
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    gk[d] = d < D ? kg[((int64_t)d * k + l) * n + coef] : 0;
    ak[d] = d < D ? ka[((int64_t)d * k + l) * n + coef] : 0;
  }
  const int64_t per = (C + gridDim.y - 1) / gridDim.y;
  const int64_t c0 = (int64_t)blockIdx.y * per;
  const int64_t c1 = c0 + per < C ? c0 + per : C;
  for (int64_t ct = c0; ct < c1; ++ct) {
    uint64_t xs[DMAX];
#pragma unroll
    for (int d = 0; d < DMAX; ++d) xs[d] = d < D ? DG[((ct * D + d) * k + l) * n + coef] : 0;
    uint64_t gh = 0, gl = 0, ah = 0, al = 0;
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
      if (d < D) {
        add128(gh, gl, __umul64hi(xs[d], gk[d]), xs[d] * gk[d]);
        add128(ah, al, __umul64hi(xs[d], ak[d]), xs[d] * ak[d]);
        if ((d & 7) == 7) {
          gl = reduce128(gh, gl, c);
          gh = 0;
          al = reduce128(ah, al, c);
          ah = 0;
        }
      }
    }
    ACC[((ct * 2 + 0) * k + l) * n + coef] = reduce128(gh, gl, c);
    ACC[((ct * 2 + 1) * k + l) * n + coef] = reduce128(ah, al, c);
  }
}

// FP64 copies of the NTT-domain key words: {signed w, w / q_l}.
__global__ void key_to_f64_kernel(const uint64_t* __restrict__ w, double2* __restrict__ f, int64_t total, int k, int logn,
                                  const LimbConst* __restrict__ lcs) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)((e >> logn) % k);
    const uint64_t q = lcs[l].q;
    const uint64_t v = w[e];
    const double s = v > q / 2 ? -(double)(q - v) : (double)v;
    f[e] = make_double2(s, s / (double)q);
  }
}

// FP64-pipe key MAC (every limb < 2^51): digits are canonical NTT outputs,
// so each product fmulq_m(x, w, w/q) has |x w/q| < 2^50 (magic rounding
// exact) and |.| < 0.75 q; sums are reduced after every 4 products (< 3.5 q).
// Both outputs' 2D key words stay in registers across the ciphertexts the
// thread walks; the next ciphertext's D digit loads are issued early.
// LEAN: only the signed key words stay in registers and the quotient comes
// from the rounded product itself (fprod: rint(RN(x w) / q), off by at most
// 1/2 + 2^-3, so products are |.| < 0.63 q and sums are reduced before every
// 6th product: < 4.3 q).  From 5 digits on the kernel runs LEAN: the key words
// take half the registers, so up to 8 digits fit 3 CTAs per SM (24 warps):
// more loads in flight, 74% -> 80% of the HBM copy peak at cfg2 (D = 7).
#ifndef FCN_KM_LEAN_FROM
#define FCN_KM_LEAN_FROM 5
#endif
// DBL: digits in and accumulators out are signed residues as raw doubles
// (the square pipeline's internal row format), |.| <= q/2 + 2^-40 q.
template <int DMAX, bool LEAN = false, bool DBL = false>
__global__ void __launch_bounds__(256, DMAX <= 8 ? 3 : 2) keymac_f64_kernel(const uint64_t* __restrict__ DG, const double2* __restrict__ kg,
                                                            const double2* __restrict__ ka, uint64_t* __restrict__ ACC,
                                                            int64_t C, int D, int k, int logn,
                                                            const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn;
  const int64_t lc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // l * n + coef
  if (lc >= (int64_t)k * n) return;
  const int l = (int)(lc >> logn);
  const int coef = (int)(lc & (n - 1));
  const double q = lcs[l].fq, qi = lcs[l].fqi;
  double2 gk[LEAN ? 1 : DMAX], ak[LEAN ? 1 : DMAX];
  double gw[LEAN ? DMAX : 1], aw[LEAN ? DMAX : 1];
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    const double2 g2 = d < D ? kg[((int64_t)d * k + l) * n + coef] : make_double2(0.0, 0.0);
    const double2 a2 = d < D ? ka[((int64_t)d * k + l) * n + coef] : make_double2(0.0, 0.0);
    if (LEAN) {
      gw[d] = g2.x;
      aw[d] = a2.x;
    } else {
      gk[d] = g2;
      ak[d] = a2;
    }
  }
  const int64_t per = (C + gridDim.y - 1) / gridDim.y;
  const int64_t c0 = (int64_t)blockIdx.y * per;
  const int64_t c1 = c0 + per < C ? c0 + per : C;
  // digits of the next PF ciphertexts in flight (PF = 2 for few digits, so
  // enough loads are outstanding per SM)
  constexpr int PF = DMAX <= 4 ? 2 : 1;
  uint64_t nx[DMAX], nx2[PF > 1 ? DMAX : 1];
#pragma unroll
  for (int d = 0; d < DMAX; ++d) nx[d] = (c0 < c1 && d < D) ? DG[((c0 * D + d) * k + l) * n + coef] : 0;
  if (PF > 1) {
#pragma unroll
    for (int d = 0; d < DMAX; ++d) nx2[d] = (c0 + 1 < c1 && d < D) ? DG[(((c0 + 1) * D + d) * k + l) * n + coef] : 0;
  }
  for (int64_t ct = c0; ct < c1; ++ct) {
    double xs[DMAX];
#pragma unroll
    for (int d = 0; d < DMAX; ++d) xs[d] = DBL ? __longlong_as_double((long long)nx[d]) : u2f(nx[d]);
    if (PF > 1) {
#pragma unroll
      for (int d = 0; d < DMAX; ++d) nx[d] = nx2[d];
      if (ct + 2 < c1) {
#pragma unroll
        for (int d = 0; d < DMAX; ++d)
          if (d < D) nx2[d] = DG[(((ct + 2) * D + d) * k + l) * n + coef];
      }
    } else if (ct + 1 < c1) {
#pragma unroll
      for (int d = 0; d < DMAX; ++d)
        if (d < D) nx[d] = DG[(((ct + 1) * D + d) * k + l) * n + coef];
    }
    double g = 0.0, a = 0.0;
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
      if (d < D) {
        if (d > 0 && (LEAN ? d % 6 == 0 : (d & 3) == 0)) {
          g = fredq(g, qi, q);
          a = fredq(a, qi, q);
        }
        if (LEAN) {
          g += fprod(xs[d], gw[d], q, qi);
          a += fprod(xs[d], aw[d], q, qi);
        } else {
          g += fmulq_m(xs[d], gk[d].x, gk[d].y, q);
          a += fmulq_m(xs[d], ak[d].x, ak[d].y, q);
        }
      }
    }
    const double gr = fredq(g, qi, q), ar = fredq(a, qi, q);
    ACC[((ct * 2 + 0) * k + l) * n + coef] = DBL ? (uint64_t)__double_as_longlong(gr) : f2u_canon(gr, q);
    ACC[((ct * 2 + 1) * k + l) * n + coef] = DBL ? (uint64_t)__double_as_longlong(ar) : f2u_canon(ar, q);
  }
}

// Shared-pair key table, coefficient domain: row (d, v) of out from the
// coefficient-domain key w [D][k][n]: v < 2 copies limb v; v = 2 + 2 (j - 2) + p
// is the centred lift of the limb-j residue reduced modulo q_p (canonical).
__global__ void pair_key_lift_kernel(const uint64_t* __restrict__ w, uint64_t* __restrict__ out, int D, int k, int logn,
                                     const LimbConst* __restrict__ lcs) {
  const int V = 2 * k - 2;
  const int64_t total = ((int64_t)D * V) << logn;
  const int n = 1 << logn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int coef = (int)(e & (n - 1));
    const int64_t r = e >> logn;
    const int v = (int)(r % V);
    const int d = (int)(r / V);
    const int j = v < 2 ? v : 2 + (v - 2) / 2;
    const int p = v & 1;
    const uint64_t x = w[(((int64_t)d * k + j) << logn) + coef];
    if (v < 2) {
      out[e] = x;
      continue;
    }
    const uint64_t qj = lcs[j].q, qp = lcs[p].q;
    // centred representative s of x mod q_j, then s mod q_p
    uint64_t y;
    if (x > qj / 2) {
      const uint64_t neg = (qj - x) % qp;  // -s mod q_p = q_p - neg
      y = neg ? qp - neg : 0;
    } else {
      y = x % qp;
    }
    out[e] = y;
  }
}

// Key MAC of the shared-pair relinearisation: virtual limb v of PairEpi's
// layout, modulus q_(v & 1).  Digits DG [C][D][2][n] (NTT domain of q_0 / q_1,
// signed doubles), keys [D][V][n]; accumulators as signed doubles:
// v < 2 -> ACCS [C][2][2][n] (the ordinary limb-0 / limb-1 sums), v >= 2 ->
// ACCP [C][2][k-2][2][n] (the two residue rows of each unit, ntt_f64_inv_pair).
// Same register scheme as keymac_f64_kernel (LEAN key words).
template <int DMAX, bool LEAN>
__global__ void __launch_bounds__(256, DMAX <= 8 ? 3 : 2)
    keymac_pair_f64_kernel(const uint64_t* __restrict__ DG, const double2* __restrict__ kg, const double2* __restrict__ ka,
                           uint64_t* __restrict__ ACCS, uint64_t* __restrict__ ACCP, int64_t C, int D, int k, int logn,
                           const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn;
  const int V = 2 * k - 2;
  const int64_t lc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // v * n + coef
  if (lc >= (int64_t)V * n) return;
  const int v = (int)(lc >> logn);
  const int coef = (int)(lc & (n - 1));
  const int p = v & 1;
  const double q = lcs[p].fq, qi = lcs[p].fqi;
  double2 gk[LEAN ? 1 : DMAX], ak[LEAN ? 1 : DMAX];
  double gw[LEAN ? DMAX : 1], aw[LEAN ? DMAX : 1];
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    const double2 g2 = d < D ? kg[((int64_t)d * V + v) * n + coef] : make_double2(0.0, 0.0);
    const double2 a2 = d < D ? ka[((int64_t)d * V + v) * n + coef] : make_double2(0.0, 0.0);
    if (LEAN) {
      gw[d] = g2.x;
      aw[d] = a2.x;
    } else {
      gk[d] = g2;
      ak[d] = a2;
    }
  }
  const int64_t per = (C + gridDim.y - 1) / gridDim.y;
  const int64_t c0 = (int64_t)blockIdx.y * per;
  const int64_t c1 = c0 + per < C ? c0 + per : C;
  uint64_t nx[DMAX];
#pragma unroll
  for (int d = 0; d < DMAX; ++d) nx[d] = (c0 < c1 && d < D) ? DG[((c0 * D + d) * 2 + p) * n + coef] : 0;
  // output rows of this virtual limb within one (ct, poly) group, and the group stride
  uint64_t* const obase = v < 2 ? ACCS + (int64_t)v * n + coef : ACCP + (int64_t)(v - 2) * n + coef;
  const int64_t gstride = (v < 2 ? 2LL : (int64_t)(V - 2)) * n;
  for (int64_t ct = c0; ct < c1; ++ct) {
    double xs[DMAX];
#pragma unroll
    for (int d = 0; d < DMAX; ++d) xs[d] = __longlong_as_double((long long)nx[d]);
    if (ct + 1 < c1) {
#pragma unroll
      for (int d = 0; d < DMAX; ++d)
        if (d < D) nx[d] = DG[(((ct + 1) * D + d) * 2 + p) * n + coef];
    }
    double g = 0.0, a = 0.0;
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
      if (d < D) {
        if (d > 0 && (LEAN ? d % 6 == 0 : (d & 3) == 0)) {
          g = fredq(g, qi, q);
          a = fredq(a, qi, q);
        }
        if (LEAN) {
          g += fprod(xs[d], gw[d], q, qi);
          a += fprod(xs[d], aw[d], q, qi);
        } else {
          g += fmulq_m(xs[d], gk[d].x, gk[d].y, q);
          a += fmulq_m(xs[d], ak[d].x, ak[d].y, q);
        }
      }
    }
    obase[(ct * 2 + 0) * gstride] = (uint64_t)__double_as_longlong(fredq(g, qi, q));
    obase[(ct * 2 + 1) * gstride] = (uint64_t)__double_as_longlong(fredq(a, qi, q));
  }
}

// Decrypt rounding m = floor((w t + (q-1)/2)/q) mod t  (fv.py:344-349).
template <int KQ, int NW>
__global__ void decrypt_round_kernel(const uint64_t* __restrict__ W, uint64_t* __restrict__ M, int64_t count, int logn,
                                     const MulCtConst* __restrict__ cc, const LimbConst* __restrict__ lcs,
                                     unsigned long long* __restrict__ fallbacks) {
  const int n = 1 << logn;
  const int k = cc->k;
  const uint64_t t = cc->t;
  const int64_t total = count << logn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ct = e >> logn;
    const int coef = (int)(e & (n - 1));
    uint64_t r[KQ];
    unsigned __int128 quo = 0;
    double G = cc->hq;
#pragma unroll
    for (int i = 0; i < KQ; ++i) {
      r[i] = 0;
      if (i < k) {
        const LimbConst& c = lcs[i];
        const uint64_t y = shoup(W[(ct * k + i) * n + coef], cc->qinv[i], cc->qinv_s[i], c.q);
        uint64_t h;
        r[i] = shoup_divmod(y, cc->tr[i], cc->tr_s[i], c.q, &h);
        quo += (unsigned __int128)h + (unsigned __int128)y * cc->tq[i];
        G += (double)r[i] * cc->rq[i];
      }
    }
    int64_t g = (int64_t)floor(G);
    const double fr = G - (double)g;
    if (fr < kEps || fr > 1.0 - kEps) {
      g = exact_frac_floor<NW>(r, k, cc, g);
      atomicAdd(fallbacks, 1ull);
    }
    quo += (unsigned __int128)g;
    M[e] = (uint64_t)(quo % t);
  }
}

// Noise budget (fv.py:356-377): the largest |centred [t w]_q| over the
// coefficients of each ciphertext's w = c0 + c1 s.  Each thread reconstructs
// its coefficients' canonical multiword values (CRT through the float64-
// estimated overflow count, corrected exactly by mw_reduce_q), centres them
// and keeps the running maximum; the block's maximum is written out and the
// host reduces the blocks (exact integers) and takes the reference's log2.
template <int KQ, int NW>
__global__ void __launch_bounds__(256) noise_max_kernel(const uint64_t* __restrict__ W, int logn,
                                                        const MulCtConst* __restrict__ cc,
                                                        const LimbConst* __restrict__ lcs, uint64_t* __restrict__ out,
                                                        int out_words) {
  __shared__ uint64_t sm[256][NW];
  const int n = 1 << logn;
  const int k = cc->k;
  const int64_t ct = blockIdx.y;
  uint64_t best[NW];
  mw_zero<NW>(best);
  for (int coef = blockIdx.x * blockDim.x + threadIdx.x; coef < n; coef += gridDim.x * blockDim.x) {
    uint64_t a[NW];
    mw_zero<NW>(a);
    double fu = 0.0;
#pragma unroll
    for (int i = 0; i < KQ; ++i) {
      if (i < k) {
        const LimbConst& c = lcs[i];
        const uint64_t x = mulmod(W[(ct * k + i) * n + coef], cc->t % c.q, c);  // [t w]_{q_i}
        const uint64_t z = shoup(x, cc->qinv[i], cc->qinv_s[i], c.q);
        fu += (double)z * cc->rq[i];
        mw_mac<NW>(a, cc->Qw[i], cc->qwords, z);
      }
    }
    mw_reduce_q<NW>(a, cc, (int64_t)floor(fu));
    uint64_t hw[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) hw[i] = i < MW_LIM ? cc->hw[i] : 0;
    if (!mw_ge<NW>(hw, a)) {  // a > (q-1)/2: |centred| = q - a
      uint64_t qa[NW];
#pragma unroll
      for (int i = 0; i < NW; ++i) qa[i] = i < MW_LIM ? cc->qw[i] : 0;
      mw_sub<NW>(qa, a);
#pragma unroll
      for (int i = 0; i < NW; ++i) a[i] = qa[i];
    }
    if (!mw_ge<NW>(best, a)) {
#pragma unroll
      for (int i = 0; i < NW; ++i) best[i] = a[i];
    }
  }
#pragma unroll
  for (int i = 0; i < NW; ++i) sm[threadIdx.x][i] = best[i];
  __syncthreads();
  for (int stride = 128; stride > 0; stride >>= 1) {
    if ((int)threadIdx.x < stride) {
      uint64_t o[NW];
#pragma unroll
      for (int i = 0; i < NW; ++i) o[i] = sm[threadIdx.x + stride][i];
      uint64_t mine[NW];
#pragma unroll
      for (int i = 0; i < NW; ++i) mine[i] = sm[threadIdx.x][i];
      if (!mw_ge<NW>(mine, o)) {
#pragma unroll
        for (int i = 0; i < NW; ++i) sm[threadIdx.x][i] = o[i];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < (unsigned)out_words)
    out[(ct * gridDim.x + blockIdx.x) * out_words + threadIdx.x] = threadIdx.x < NW ? sm[0][threadIdx.x] : 0;
}

// ------------------------------------------------------ host constants

static Big big_prod(const std::vector<uint64_t>& v, int skip = -1) {
  Big r(1);
  for (int i = 0; i < (int)v.size(); ++i)
    if (i != skip) r = r.mul_small(v[i]);
  return r;
}

static void store_words(const Big& b, uint64_t* dst, int cap) {
  for (int i = 0; i < cap; ++i) dst[i] = b.word(i);
}

static int build_mulct_const(const fcn_ctx* x, uint64_t t, MulCtConst* mc) {
  memset(mc, 0, sizeof(*mc));
  const int k = x->k, m = x->m, K = k + m;
  mc->k = k;
  mc->m = m;
  mc->K = K;
  mc->D = x->ell + 1;
  mc->w = x->log2_beta;
  mc->t = t;
  std::vector<uint64_t> ext = x->primes;
  ext.insert(ext.end(), x->aux.begin(), x->aux.end());
  const Big q = big_prod(x->primes);
  const Big P = big_prod(x->aux);
  mc->qwords = (int)q.w.size();
  store_words(q, mc->qw, MW_LIM);
  store_words(q.shr1(), mc->hw, MW_LIM);
  const double qd = q.to_double();
  mc->hq = 0.5 - 0.5 / qd;
  // lift
  for (int i = 0; i < k; ++i) {
    const uint64_t qi = x->primes[i];
    const Big Qi = big_prod(x->primes, i);
    store_words(Qi, mc->Qw[i], MW_LIM);
    const uint64_t qm = Qi.mod_small(qi);
    mc->qinv[i] = h_powmod(qm, qi - 2, qi);
    mc->qinv_s[i] = h_shoup(mc->qinv[i], qi);
    mc->rq[i] = 1.0 / (double)qi;
  }
  for (int j = 0; j < m; ++j) {
    const uint64_t p = x->aux[j];
    for (int i = 0; i < k; ++i) {
      const uint64_t c = big_prod(x->primes, i).mod_small(p);
      mc->lc[j][i] = c;
      mc->lc_s[j][i] = h_shoup(c, p);
    }
    const uint64_t qp = q.mod_small(p);
    for (int v = 0; v <= k + 1; ++v) mc->lvq[j][v] = (p - h_mulmod(qp, (uint64_t)v, p)) % p;
  }
  // rescale
  const Big B = q.mul(P);
  const Big tP = P.mul_small(t);
  for (int j = 0; j < K; ++j) {
    const uint64_t b = ext[j];
    const uint64_t bm = big_prod(ext, j).mod_small(b);
    mc->binv[j] = h_powmod(bm, b - 2, b);
    mc->binv_s[j] = h_shoup(mc->binv[j], b);
    mc->rb[j] = 1.0 / (double)b;
  }
  (void)B;
  std::vector<Big> alpha(k);
  for (int j = 0; j < k; ++j) {
    uint64_t rem;
    alpha[j] = tP.div_small(x->primes[j], &rem);
    mc->beta[j] = rem;
    mc->beta_s[j] = h_shoup(rem, x->primes[j]);
  }
  std::vector<Big> tPp(m);
  for (int j = 0; j < m; ++j) {
    uint64_t rem;
    tPp[j] = tP.div_small(x->aux[j], &rem);
    if (rem) return set_error(FCN_ERR_PARAM, "internal: aux prime does not divide tP");
  }
  for (int i = 0; i < k; ++i) {
    const uint64_t qi = x->primes[i];
    for (int j = 0; j < K; ++j) {
      const uint64_t c = j < k ? alpha[j].mod_small(qi) : tPp[j - k].mod_small(qi);
      mc->rc[i][j] = c;
      mc->rc_s[i][j] = h_shoup(c, qi);
    }
    const uint64_t tpm = tP.mod_small(qi);
    for (int v = 0; v <= K + 1; ++v) mc->rvt[i][v] = (qi - h_mulmod(tpm, (uint64_t)v, qi)) % qi;
    // decrypt
    mc->tr[i] = t % qi;
    mc->tq[i] = t / qi;
    mc->tr_s[i] = h_shoup(mc->tr[i], qi);
    // digits: 2^(64 m) mod q_i
    for (int mm = 0; mm < 4; ++mm) {
      uint64_t pw = 1 % qi;
      for (int s = 0; s < mm; ++s) pw = (uint64_t)(((unsigned __int128)pw << 64) % qi);
      mc->dpw[i][mm] = pw;
      mc->dpw_s[i][mm] = h_shoup(pw, qi);
    }
    // add_pt
    uint64_t dr;
    const Big delta = q.div_small(t, &dr);
    mc->delta[i] = delta.mod_small(qi);
    mc->delta_s[i] = h_shoup(mc->delta[i], qi);
  }
  uint64_t qmin = ~0ull;
  for (uint64_t qi : x->primes) qmin = qi < qmin ? qi : qmin;
  mc->direct = (mc->w < 64 && ((1ull << mc->w) <= qmin)) ? 1 : 0;
  mc->dwords = (mc->w + 63) / 64;
  if (mc->dwords > 3) return set_error(FCN_ERR_PARAM, "log2(beta) = %d exceeds the supported 192 bits", mc->w);
  return FCN_OK;
}

}  // namespace fcn

using namespace fcn;

// ----------------------------------------------------------------- C ABI

static bool f64_lift_rescale(const fcn_ctx* x);
static double h_signed(uint64_t w, uint64_t q) { return w > q / 2 ? -(double)(q - w) : (double)w; }

// Shared-pair relinearisation (PairEpi): usable when the digits are plain
// integers below every limb (beta <= q_min), every q-limb runs the FP64
// kernels, the key-switching sums |V_j| <= D n (beta - 1) (q_j - 1) / 2 stay
// below 0.45 q_0 q_1 (so the two-residue CRT is exact, with margin for the
// 2^-40 slack of the centred residues), and 2D + 4k - 4 transformed rows per
// ciphertext beat the direct k (D + 2).  FCN_PAIR_RELIN=0 disables it.
static void pair_relin_setup(fcn_ctx* x) {
  x->pair = false;
  const char* ev = getenv("FCN_PAIR_RELIN");
  if (ev && ev[0] == '0') return;
  const int k = x->k, D = x->ell + 1, w = x->log2_beta, n = x->n;
  if (!x->fp || k < 3 || k > kPairLimbs || D > 12 || x->logn < 10 || x->logn > 14) return;
  if (!f64_lift_rescale(x)) return;  // the square pipeline's signed-double rows come from the FP64 lift / rescale
  uint64_t qmin = ~0ull, qmax = 0;
  for (uint64_t q : x->primes) {
    qmin = q < qmin ? q : qmin;
    qmax = q > qmax ? q : qmax;
  }
  if (w >= 64 || (1ull << w) > qmin || qmax / qmin >= 4) return;
  if (ntt_family(x->ext, k, 0) != 2) return;
  if (2 * D + 4 * k - 4 >= k * (D + 2)) return;
  const uint64_t q0 = x->primes[0], q1 = x->primes[1];
  const long double vmax = (long double)D * n * (long double)((1ull << w) - 1) * ((long double)(qmax - 1) / 2);
  if (vmax > 0.45L * (long double)q0 * (long double)q1) return;
  const uint64_t i01 = h_powmod(q0 % q1, q1 - 2, q1);
  x->pair_inv01 = h_signed(i01, q1);
  x->pair_inv01q = x->pair_inv01 / (double)q1;
  for (int j = 0; j < k; ++j) {
    const uint64_t qj = x->primes[j];
    x->pair_c0[j] = h_signed(q0 % qj, qj);
    x->pair_c0q[j] = x->pair_c0[j] / (double)qj;
  }
  x->pair = true;
}

extern "C" int fcn_ctx_create(int device, int n, int k, const uint64_t* primes, int n_lanes, const uint64_t* t_lanes,
                              int log2_beta, fcn_ctx** out) {
  if (!out || !primes || !t_lanes || k <= 0 || n_lanes <= 0) return set_error(FCN_ERR_ARG, "bad context arguments");
  if (k > KQ_LIM) return set_error(FCN_ERR_PARAM, "at most %d ciphertext limbs are supported", KQ_LIM);
  if (n_lanes > LANE_LIM) return set_error(FCN_ERR_PARAM, "at most %d plaintext lanes", LANE_LIM);
  if (log2_beta < 1 || log2_beta > 190) return set_error(FCN_ERR_PARAM, "log2(beta) must be in [1, 190]");
  fcn_ctx* x = new fcn_ctx();
  x->device = device;
  x->n = n;
  x->k = k;
  x->log2_beta = log2_beta;
  x->n_lanes = n_lanes;
  x->primes.assign(primes, primes + k);
  x->lanes.assign(t_lanes, t_lanes + n_lanes);
  for (int i = 0; i < k; ++i)
    for (int j = i + 1; j < k; ++j)
      if (primes[i] == primes[j]) {
        delete x;
        return set_error(FCN_ERR_PARAM, "duplicate limb prime");
      }
  const Big q = big_prod(x->primes);
  for (uint64_t t : x->lanes) {
    if (t < 2) {
      delete x;
      return set_error(FCN_ERR_PARAM, "plaintext modulus must be >= 2");
    }
    uint64_t r;
    const Big d = q.div_small(t, &r);
    if (d.bits() <= 16) {
      delete x;
      return set_error(FCN_ERR_PARAM, "ciphertext modulus too small for lane t=%llu", (unsigned long long)t);
    }
  }
  // ell = max e with beta^e <= q  (fv.py:78-85)
  x->ell = (q.bits() - 1) / log2_beta;
  // Auxiliary base.  The reference scans find_ntt_primes(n, need//54 + 1,
  // bits=55, exclude=q) (fv.py:99-107); the base only has to make the
  // extended-base CRT of the tensor exact, which needs P > 2nq.  We take
  // the first NTT primes above 2^50 (ascending scan, limb primes excluded),
  // the smallest count giving P >= 8nq, so |T|/B <= 1/16 (section 5 of
  // DESIGN.md); outputs do not depend on the choice.  Primes just above 2^50
  // keep every extended-base limb on the FP64 kernels (q < 2^51) and let the
  // FP64 NTT reduce once per transform instead of four times (ntt_f64.cuh).
  int nb = 0;
  while ((1 << nb) <= n) ++nb;
  const int need = nb + q.bits() + 3;
  const int count = (need + 49) / 50;
  const uint64_t step = 2ull * (uint64_t)n;
  uint64_t p = ((1ull << 50) / step) * step + 1;
  while ((int)x->aux.size() < count && p < (1ull << 51) - step) {
    p += step;
    bool skip = false;
    for (uint64_t qq : x->primes) skip |= qq == p;
    if (!skip && h_is_prime(p)) x->aux.push_back(p);
  }
  if ((int)x->aux.size() < count) {
    delete x;
    return set_error(FCN_ERR_PARAM, "not enough auxiliary NTT primes in (2^50, 2^51)");
  }
  x->m = count;
  if (k + count > KE_LIM) {
    delete x;
    return set_error(FCN_ERR_PARAM, "extended base of %d limbs exceeds %d", k + count, KE_LIM);
  }
  std::vector<uint64_t> ext = x->primes;
  ext.insert(ext.end(), x->aux.begin(), x->aux.end());
  int rc = fcn_ring_create(device, n, (int)ext.size(), ext.data(), &x->ext);
  if (rc) {
    delete x;
    return rc;
  }
  x->logn = x->ext->logn;
  {
    const char* ev = getenv("FCN_NTT_INT");  // A/B switch: integer kernels only
    x->fp = x->ext->fp_ok && !(ev && ev[0] == '1');
  }
  if (x->fp && !f64_lift_rescale(x) && !getenv("FCN_QUIET"))
    fprintf(stderr,
            "[libfcn] k=%d q-limbs + m=%d auxiliary limbs has no exact-size FP64 lift/rescale instantiation "
            "(csrc/fv.cu lift_or_rescale): mul_ct runs the integer lift/rescale kernels\n",
            k, x->m);
  std::vector<MulCtConst> host(n_lanes);
  for (int l = 0; l < n_lanes; ++l) {
    rc = build_mulct_const(x, x->lanes[l], &host[l]);
    if (rc) {
      fcn_ctx_destroy(x);
      return rc;
    }
  }
  x->host_mc = host;
  DeviceGuard g(device);
  cudaError_t e = cudaMalloc(&x->d_mc, sizeof(MulCtConst) * n_lanes);
  if (e == cudaSuccess) e = cudaMemcpy(x->d_mc, host.data(), sizeof(MulCtConst) * n_lanes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&x->d_fallbacks, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(x->d_fallbacks, 0, sizeof(unsigned long long));
  if (e == cudaSuccess && x->fp) {
    // twist_l[j] (B/b_l)^-1 for the tensor's inverse NTT (the rescale then
    // starts from y_j = T_j (B/b_l)^-1 directly, fv.py:473-490)
    const int K = (int)ext.size();
    std::vector<double2> tw((size_t)K * n);
    for (int l = 0; l < K; ++l) {
      const uint64_t b = ext[l];
      const uint64_t iroot = h_powmod(x->ext->roots[l], b - 2, b);
      const uint64_t ninv = h_powmod((uint64_t)n % b, b - 2, b);
      uint64_t w = h_mulmod(ninv, host[0].binv[l], b);
      for (int j = 0; j < n; ++j) {
        const double ws = w > b / 2 ? -(double)(b - w) : (double)w;
        tw[(size_t)l * n + j] = make_double2(ws, ws / (double)b);
        w = h_mulmod(w, iroot, b);
      }
    }
    e = cudaMalloc(&x->d_ftwist_binv, sizeof(double2) * tw.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(x->d_ftwist_binv, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    fcn_ctx_destroy(x);
    return check_cuda(e, "fcn_ctx_create upload");
  }
  pair_relin_setup(x);
  *out = x;
  return FCN_OK;
}

extern "C" int fcn_ctx_destroy(fcn_ctx* x) {
  if (!x) return FCN_OK;
  {
    DeviceGuard g(x->device);
    cudaFree(x->d_mc);
    cudaFree(x->d_fallbacks);
    cudaFree(x->d_ftwist_binv);
    for (auto& kv : x->ftwist_c2) cudaFree(kv.second);
  }
  fcn_ring_destroy(x->ext);
  delete x;
  return FCN_OK;
}

extern "C" int fcn_ctx_ring(const fcn_ctx* x, const fcn_ring** out) {
  if (!x || !out) return set_error(FCN_ERR_ARG, "null argument");
  *out = x->ext;
  return FCN_OK;
}

extern "C" int fcn_ctx_query(const fcn_ctx* x, int what, int64_t* value) {
  if (!x || !value) return set_error(FCN_ERR_ARG, "null argument");
  switch (what) {
    case 0: *value = x->n; break;
    case 1: *value = x->k; break;
    case 2: *value = x->m; break;
    case 3: *value = x->ell; break;
    case 4: *value = x->n_lanes; break;
    case 5: *value = x->log2_beta; break;
    case 6: *value = f64_lift_rescale(x) ? 1 : 0; break;
    case 7: *value = x->pair ? 1 : 0; break;
    default: return set_error(FCN_ERR_ARG, "unknown query %d", what);
  }
  return FCN_OK;
}

extern "C" int fcn_ctx_aux_primes(const fcn_ctx* x, uint64_t* out_m) {
  if (!x || !out_m) return set_error(FCN_ERR_ARG, "null argument");
  for (int j = 0; j < x->m; ++j) out_m[j] = x->aux[j];
  return FCN_OK;
}

extern "C" int fcn_ctx_fallback_count(const fcn_ctx* x, int64_t* value) {
  if (!x || !value) return set_error(FCN_ERR_ARG, "null argument");
  DeviceGuard g(x->device);
  unsigned long long v = 0;
  FCN_CUDA(cudaMemcpy(&v, x->d_fallbacks, sizeof(v), cudaMemcpyDeviceToHost));
  *value = (int64_t)v;
  return FCN_OK;
}

extern "C" int fcn_keys_create(const fcn_ctx* x, const uint64_t* a, const uint64_t* g, fcn_keys** out) {
  if (!x || !a || !g || !out) return set_error(FCN_ERR_ARG, "null argument");
  fcn_keys* kk = new fcn_keys();
  kk->device = x->device;
  kk->D = x->ell + 1;
  kk->k = x->k;
  kk->n = x->n;
  const size_t words = (size_t)kk->D * kk->k * kk->n;
  DeviceGuard gd(x->device);
  cudaError_t e = cudaMalloc(&kk->d_g, words * 8);
  if (e == cudaSuccess) e = cudaMalloc(&kk->d_a, words * 8);
  if (e == cudaSuccess) e = cudaMemcpy(kk->d_g, g, words * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(kk->d_a, a, words * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    fcn_keys_destroy(kk);
    return check_cuda(e, "fcn_keys_create upload");
  }
  int rc = FCN_OK;
  if (x->pair) {
    // shared-pair tables from the coefficient-domain words (before the in-place transforms below)
    const int V = 2 * kk->k - 2;
    const size_t pwords = (size_t)kk->D * V * kk->n;
    uint64_t* tmp = nullptr;
    e = cudaMalloc(&tmp, pwords * 8);
    if (e == cudaSuccess) e = cudaMalloc(&kk->d_pg, pwords * sizeof(double2));
    if (e == cudaSuccess) e = cudaMalloc(&kk->d_pa, pwords * sizeof(double2));
    for (int which = 0; which < 2 && e == cudaSuccess && !rc; ++which) {
      pair_key_lift_kernel<<<grid_for((int64_t)pwords, 256), 256>>>(which ? kk->d_a : kk->d_g, tmp, kk->D, kk->k, x->logn,
                                                                    x->ext->d_lc);
      e = cudaGetLastError();
      if (e == cudaSuccess) rc = launch_ntt(x->ext, tmp, (int64_t)kk->D * V, 2, 0, true, 0);
      if (e == cudaSuccess && !rc) {
        key_to_f64_kernel<<<grid_for((int64_t)pwords, 256), 256>>>(tmp, which ? kk->d_pa : kk->d_pg, (int64_t)pwords, 2,
                                                                   x->logn, x->ext->d_lc);
        e = cudaGetLastError();
      }
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(tmp);
    if (e != cudaSuccess) rc = check_cuda(e, "fcn_keys_create shared-pair tables");
  }
  if (!rc) rc = launch_ntt(x->ext, kk->d_g, (int64_t)kk->D * kk->k, kk->k, 0, true, 0);
  if (!rc) rc = launch_ntt(x->ext, kk->d_a, (int64_t)kk->D * kk->k, kk->k, 0, true, 0);
  if (!rc && x->fp && kk->D <= 12) {
    e = cudaMalloc(&kk->d_fg, words * sizeof(double2));
    if (e == cudaSuccess) e = cudaMalloc(&kk->d_fa, words * sizeof(double2));
    if (e != cudaSuccess) {
      rc = check_cuda(e, "fcn_keys_create fp64 copies");
    } else {
      key_to_f64_kernel<<<grid_for((int64_t)words, 256), 256>>>(kk->d_g, kk->d_fg, (int64_t)words, kk->k, x->logn,
                                                                x->ext->d_lc);
      key_to_f64_kernel<<<grid_for((int64_t)words, 256), 256>>>(kk->d_a, kk->d_fa, (int64_t)words, kk->k, x->logn,
                                                                x->ext->d_lc);
      e = cudaGetLastError();
      if (e != cudaSuccess) rc = check_cuda(e, "key_to_f64_kernel");
    }
  }
  if (!rc) {
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = check_cuda(e, "fcn_keys_create ntt");
  }
  if (rc) {
    fcn_keys_destroy(kk);
    return rc;
  }
  *out = kk;
  return FCN_OK;
}

extern "C" int fcn_keys_destroy(fcn_keys* kk) {
  if (!kk) return FCN_OK;
  {
    DeviceGuard g(kk->device);
    cudaFree(kk->d_g);
    cudaFree(kk->d_a);
    cudaFree(kk->d_fg);
    cudaFree(kk->d_fa);
    cudaFree(kk->d_pg);
    cudaFree(kk->d_pa);
  }
  delete kk;
  return FCN_OK;
}

extern "C" int fcn_add_plain_terms(const fcn_ctx* x, int lane, uint64_t* d_cts, int64_t n_terms, const int32_t* d_ct_index,
                                   const int32_t* d_pos, const int64_t* d_coef, void* stream) {
  if (!x || lane < 0 || lane >= x->n_lanes) return set_error(FCN_ERR_ARG, "bad context or lane");
  if (n_terms <= 0) return FCN_OK;
  if (!d_cts || !d_ct_index || !d_pos || !d_coef) return set_error(FCN_ERR_ARG, "null argument");
  DeviceGuard g(x->device);
  const int64_t total = n_terms * x->k;
  add_plain_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(d_cts, n_terms, d_ct_index, d_pos, d_coef, x->k,
                                                                          x->logn, x->d_mc + lane, x->ext->d_lc);
  FCN_LAUNCH_CHECK("add_plain_kernel");
  return FCN_OK;
}

extern "C" int fcn_linear_mac(const fcn_ctx* x, const uint64_t* d_in0, int64_t n_in0, const uint64_t* d_in1, int64_t n_in1,
                              const int32_t* d_rowptr, const int32_t* d_col, const int32_t* d_rot, const int64_t* d_coef,
                              uint64_t* d_out, int64_t n_out, void* stream) {
  return fcn_linear_mac_ex(x, d_in0, n_in0, d_in1, n_in1, d_rowptr, d_col, d_rot, d_coef, d_out, n_out, 0, 0, stream);
}

extern "C" int fcn_linear_mac_ex(const fcn_ctx* x, const uint64_t* d_in0, int64_t n_in0, const uint64_t* d_in1,
                                 int64_t n_in1, const int32_t* d_rowptr, const int32_t* d_col, const int32_t* d_rot,
                                 const int64_t* d_coef, uint64_t* d_out, int64_t n_out, int no_rot, uint64_t max_abs_coef,
                                 void* stream) {
  uint64_t* outs[1] = {d_out};
  return fcn_linear_mac_multi(x, d_in0, n_in0, d_in1, n_in1, d_rowptr, d_col, d_rot, d_coef, outs, 1, n_out, no_rot,
                              max_abs_coef, stream);
}

static bool mac_sgn_enabled();

extern "C" int fcn_linear_mac_multi(const fcn_ctx* x, const uint64_t* d_in0, int64_t n_in0, const uint64_t* d_in1,
                                    int64_t n_in1, const int32_t* d_rowptr, const int32_t* d_col, const int32_t* d_rot,
                                    const int64_t* d_coef, uint64_t* const* d_outs, int n_dst, int64_t n_out, int no_rot,
                                    uint64_t max_abs_coef, void* stream) {
  if (!x) return set_error(FCN_ERR_ARG, "null context");
  if (n_out <= 0) return FCN_OK;
  if (n_dst < 1 || n_dst > kMaxFanout || !d_outs) return set_error(FCN_ERR_ARG, "1..%d destinations", kMaxFanout);
  Fanout F;
  F.n = n_dst;
  for (int d = 0; d < n_dst; ++d) {
    if (!d_outs[d]) return set_error(FCN_ERR_ARG, "null destination %d", d);
    F.dst[d] = d_outs[d];
  }
  if (!d_rowptr || (n_in0 > 0 && !d_in0) || (n_in1 > 0 && !d_in1)) return set_error(FCN_ERR_ARG, "null argument");
  if (n_out > 65535) return set_error(FCN_ERR_ARG, "at most 65535 outputs per launch");
  DeviceGuard g(x->device);
  const int threads = 256;
  // lazy 64-bit accumulation: fold * max|c| * q_max + 4 q_max < 2^64
  uint64_t qmax = 0;
  for (uint64_t q : x->primes) qmax = q > qmax ? q : qmax;
  int fold = 0;
  if (no_rot && max_abs_coef > 0 && max_abs_coef < (1ull << 32)) {
    const unsigned __int128 room = ((unsigned __int128)1 << 64) - 4 * (unsigned __int128)qmax;
    const unsigned __int128 per = (unsigned __int128)qmax * max_abs_coef;
    const unsigned __int128 f = room / per;
    fold = f > 1024 ? 1024 : (int)f;
  }
  // SMALL variant (every limb in [2^34, 2^56)): sums bounded by 2^62 so one
  // high-word quotient reduces them (reduce_small) instead of a Shoup product
  bool small = fold >= 2;
  for (uint64_t q : x->primes) small &= q >= (1ull << 34) && q < (1ull << 56);
  int fold_small = 0;
  if (small) {
    const unsigned __int128 f = (((unsigned __int128)1 << 62) - qmax) / ((unsigned __int128)qmax * max_abs_coef);
    fold_small = f > 1024 ? 1024 : (int)f;
    small = fold_small >= 2;
  }
  // signed single-accumulator variant: |acc| < 2^60
  int fold_sgn = 0;
  if (small) {
    const unsigned __int128 f = (((unsigned __int128)1 << 60) - qmax) / ((unsigned __int128)qmax * max_abs_coef);
    fold_sgn = f > 1024 ? 1024 : (int)f;
  }
  const bool sgn = small && fold_sgn >= 4 && mac_sgn_enabled();
  if (fold >= 2 && x->n >= 4) {
    // blockIdx.x (fastest) walks outputs, so the CTAs resident at any time
    // (~148 x 8) share one (row, coefficient tile): that tile's slice of
    // every input stays in L2 while all outputs referencing it are summed.
    // The tile (4 residues per thread) shrinks so n_in slices fit in ~48 MB.
    const int64_t n_in_all = n_in0 + n_in1;
    constexpr int NR = MAC_ROWS;  // rows (c0, c1 of one limb) per thread
    int th = threads;
    while (th > 32 && n_in_all * th * 4 * 8 * NR > (48ll << 20)) th >>= 1;
    const int per_cta = th * 4;
    const int gy = (x->n + per_cta - 1) / per_cta, gz = 2 * x->k / NR;
    int64_t gx = 148LL * 8 * MAC_WAVES / 4;
    if (gx > n_out) gx = n_out;
    if (gx < 1) gx = 1;
    dim3 grid((unsigned)gx, gy, gz);
    if (sgn)
      mac_fast_kernel<true, NR, true><<<grid, th, 0, (cudaStream_t)stream>>>(
          d_in0, n_in0, d_in1, d_rowptr, d_col, d_coef, F, x->logn, x->k, x->ext->d_lc, fold_sgn, (int)n_out);
    else if (small)
      mac_fast_kernel<true, NR><<<grid, th, 0, (cudaStream_t)stream>>>(d_in0, n_in0, d_in1, d_rowptr, d_col, d_coef, F,
                                                                     x->logn, x->k, x->ext->d_lc, fold_small, (int)n_out);
    else
      mac_fast_kernel<false, NR><<<grid, th, 0, (cudaStream_t)stream>>>(d_in0, n_in0, d_in1, d_rowptr, d_col, d_coef, F,
                                                                      x->logn, x->k, x->ext->d_lc, fold, (int)n_out);
    FCN_LAUNCH_CHECK("mac_fast_kernel");
    return FCN_OK;
  }
  const int per_cta = threads * 2;
  dim3 grid((x->n + per_cta - 1) / per_cta, (unsigned)n_out, 2 * x->k);
  mac_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(d_in0, n_in0, d_in1, d_rowptr, d_col, d_rot, d_coef, F, x->logn,
                                                         x->k, x->ext->d_lc);
  FCN_LAUNCH_CHECK("mac_kernel");
  return FCN_OK;
}

// workspace per ciphertext in words: EA, EB (2K each), T (3K), R01 (2k),
// DGN (D k), ACC (2k), raw digit rows (D)
// ---- tensor-core linear layer (csrc/mac_tc.cu)

static int tc_planes(const fcn_ctx* x) {
  uint64_t qmax = 0;
  for (uint64_t q : x->primes) qmax = q > qmax ? q : qmax;
  const int bits = bitlen64(qmax);
  return (bits + 7) / 8;
}

extern "C" int fcn_tc_planes(const fcn_ctx* x) {
  if (!x) return set_error(FCN_ERR_ARG, "null context");
  const int P = tc_planes(x);
  return (P >= 5 && P <= 8) ? P : 0;
}

extern "C" size_t fcn_tc_planes_bytes(const fcn_ctx* x, int64_t count) {
  if (!x || count <= 0) return 0;
  return (size_t)count * (size_t)tc_planes(x) * (size_t)tc_plane_pitch(2LL * x->k * x->n);
}

extern "C" int fcn_split_planes(const fcn_ctx* x, const uint64_t* d_in, int64_t count, uint8_t* d_planes, void* stream) {
  if (!x) return set_error(FCN_ERR_ARG, "null context");
  if (count <= 0) return FCN_OK;
  if (!d_in || !d_planes) return set_error(FCN_ERR_ARG, "null buffer");
  const int P = tc_planes(x);
  if (P < 5 || P > 8) return set_error(FCN_ERR_PARAM, "byte planes need limbs in [2^32, 2^64)");
  DeviceGuard g(x->device);
  return launch_split_planes(d_in, count, 2LL * x->k * x->n, P, d_planes, (cudaStream_t)stream);
}

extern "C" int fcn_linear_mac_tc(const fcn_ctx* x, const uint8_t* d_planes, int64_t n_in, int64_t n_groups,
                                 const int32_t* d_groups, const int32_t* d_kidx, const int32_t* d_rows,
                                 const int8_t* d_wimg, uint64_t* const* d_outs, int n_dst, int64_t row_lo,
                                 int64_t row_hi, void* stream) {
  if (!x) return set_error(FCN_ERR_ARG, "null context");
  if (n_groups <= 0 || row_hi <= row_lo) return FCN_OK;
  if (n_dst < 1 || n_dst > kMaxFanout || !d_outs) return set_error(FCN_ERR_ARG, "1..%d destinations", kMaxFanout);
  if (!d_planes || !d_groups || !d_kidx || !d_rows || !d_wimg) return set_error(FCN_ERR_ARG, "null argument");
  if (n_in <= 0) return set_error(FCN_ERR_ARG, "no inputs");
  const int P = tc_planes(x);
  if (P < 5 || P > 8) return set_error(FCN_ERR_PARAM, "byte planes need limbs in [2^32, 2^64)");
  TcLaunch a;
  a.planes = d_planes;
  a.cols = 2LL * x->k * x->n;
  a.planes_n = P;
  a.n_groups = n_groups;
  a.groups = reinterpret_cast<const TcGroup*>(d_groups);
  a.kidx = d_kidx;
  a.rows = d_rows;
  a.wimg = d_wimg;
  a.out.n = n_dst;
  for (int d = 0; d < n_dst; ++d) {
    if (!d_outs[d]) return set_error(FCN_ERR_ARG, "null destination %d", d);
    a.out.dst[d] = d_outs[d];
  }
  a.row_lo = row_lo;
  a.row_hi = row_hi;
  a.logn = x->logn;
  a.k = x->k;
  a.lcs = x->ext->d_lc;
  DeviceGuard g(x->device);
  return launch_mac_tc(a, (cudaStream_t)stream);
}

static int64_t mulct_words_per_ct(const fcn_ctx* x) {
  const int64_t K = x->k + x->m, k = x->k, D = x->ell + 1;
  return (2 * K + 2 * K + 3 * K + 2 * k + D * k + 2 * k + D) * (int64_t)x->n;
}

extern "C" size_t fcn_mul_ct_workspace_bytes(const fcn_ctx* x, int64_t chunk) {
  if (!x || chunk <= 0) return 0;
  return (size_t)(mulct_words_per_ct(x) * chunk * 8);
}

// signed representative in (-q/2, q/2] as a double (q < 2^51: exact)

template <int KQ, int KA>
static LiftP<KQ, KA> make_lift_params(const fcn_ctx* x, const MulCtConst& mc) {
  LiftP<KQ, KA> P;
  memset(&P, 0, sizeof(P));
  P.k = x->k;
  P.m = x->m;
  P.K = x->k + x->m;
  const Big q = big_prod(x->primes);
  for (int i = 0; i < x->k; ++i) {
    P.q[i] = x->primes[i];
    P.nq[i] = (uint64_t)0 - x->primes[i];
    P.qinv[i] = mc.qinv[i];
    P.qinv_s[i] = mc.qinv_s[i];
    P.rq[i] = mc.rq[i];
    P.fq[i] = (double)x->primes[i];
    P.fqinv[i] = h_signed(mc.qinv[i], x->primes[i]);
    P.fqinvq[i] = P.fqinv[i] / P.fq[i];
  }
  for (int j = 0; j < x->m; ++j) {
    const uint64_t pj = x->aux[j];
    P.fp[j] = (double)pj;
    P.fpi[j] = 1.0 / (double)pj;
    for (int i = 0; i < x->k; ++i) {
      P.flc[j][i] = h_signed(mc.lc[j][i], pj);
      P.flcq[j][i] = P.flc[j][i] / (double)pj;
    }
    P.p[j] = pj;
    P.np[j] = (uint64_t)0 - pj;
    P.p_one_s[j] = h_shoup(1, pj);
    for (int i = 0; i < x->k; ++i) {
      P.lc[j][i] = mc.lc[j][i];
      P.lc_s[j][i] = mc.lc_s[j][i];
    }
    const uint64_t qp = q.mod_small(pj);
    P.nqp[j] = (pj - qp) % pj;
    P.nqp_s[j] = h_shoup(P.nqp[j], pj);
    P.fnqp[j] = h_signed(P.nqp[j], pj);
    P.fnqpq[j] = P.fnqp[j] / (double)pj;
  }
  return P;
}

template <int KQ, int KE>
static RescaleP<KQ, KE> make_rescale_params(const fcn_ctx* x, const MulCtConst& mc) {
  RescaleP<KQ, KE> P;
  memset(&P, 0, sizeof(P));
  const int k = x->k, K = x->k + x->m;
  P.k = k;
  P.K = K;
  P.D = mc.D;
  P.w = mc.w;
  P.direct = mc.direct;
  P.dwords = mc.dwords;
  for (int j = 0; j < K; ++j) {
    P.q[j] = j < k ? x->primes[j] : x->aux[j - k];
    P.nq[j] = (uint64_t)0 - P.q[j];
    P.binv[j] = mc.binv[j];
    P.binv_s[j] = mc.binv_s[j];
    P.rb[j] = mc.rb[j];
    P.fb[j] = (double)P.q[j];
    P.fbinv[j] = h_signed(mc.binv[j], P.q[j]);
    P.fbinvq[j] = P.fbinv[j] / (double)P.q[j];
  }
  for (int i = 0; i < k; ++i) {
    const uint64_t qi = x->primes[i];
    P.one_s[i] = h_shoup(1, qi);
    P.rq[i] = mc.rq[i];
    P.beta[i] = mc.beta[i];
    P.beta_s[i] = mc.beta_s[i];
    P.qinv[i] = mc.qinv[i];
    P.qinv_s[i] = mc.qinv_s[i];
    for (int j = 0; j < K; ++j) {
      P.rc[i][j] = mc.rc[i][j];
      P.rc_s[i][j] = mc.rc_s[i][j];
    }
    P.ntp[i] = mc.rvt[i][1];  // (-tP) mod q_i
    P.ntp_s[i] = h_shoup(P.ntp[i], qi);
    P.fq[i] = (double)qi;
    P.fqi[i] = 1.0 / (double)qi;
    P.fbeta[i] = (double)mc.beta[i];
    P.fbetaq[i] = (double)mc.beta[i] / (double)qi;
    P.fntp[i] = h_signed(P.ntp[i], qi);
    P.fntpq[i] = P.fntp[i] / (double)qi;
    for (int j = 0; j < K; ++j) {
      P.frc[i][j] = h_signed(mc.rc[i][j], qi);
      P.frcq[i][j] = P.frc[i][j] / (double)qi;
    }
    for (int mm = 0; mm < 3; ++mm) {
      P.dpw[i][mm] = mc.dpw[i][mm];
      P.dpw_s[i][mm] = mc.dpw_s[i][mm];
    }
  }
  return P;
}

struct ActArgs {
  bool on = false;
  int64_t c2 = 1, c1 = 0;
  const uint64_t* lin = nullptr;
  bool applied = false;  // set when the rescale kernel folded it into R01
  bool prescaled = false;  // the tensor INTT already multiplied by (B/b_j)^-1 (FP64 rescale only)
  bool dbl_in = false;     // ... and left the rows as signed doubles
};

// Products accumulated between reductions in the FP64 lift / rescale: a
// product a w mod q with |a| <= 0.75 b, |w| <= q/2 (b, q < 2^51) is
// |.| <= (1/2 + 0.75 b 2^-53) q, a reduced sum |.| <= q/2, and a sum starts
// at <= q; 12 products are allowed when 1/2 + 12 p and 1 + 11 p stay below
// 2^53 / q for the largest prime (limbs just above 2^50), else 4.
static int f64_product_period(const fcn_ctx* x) {
  uint64_t mx = 0;
  for (uint64_t v : x->primes) mx = v > mx ? v : mx;
  for (uint64_t v : x->aux) mx = v > mx ? v : mx;
  const double p = 0.5 + 0.75 * (double)mx * 0x1p-53 + 0x1p-20;
  const double lim = 0x1p53 / ((double)mx + 1.0) * (1.0 - 1e-9);
  return (0.5 + 12 * p < lim && 1.0 + 11 * p < lim) ? 12 : 4;
}

template <int KQ, int KE>
static int run_lift_rescale(bool lift, const fcn_ctx* x, int lane, const uint64_t* in, uint64_t* out, int64_t cnt,
                            uint64_t* R01, uint64_t* DG, cudaStream_t st, ActArgs* act, bool* compact,
                            const int* lift_mode) {
  const bool f64 = x->fp && x->k == KQ && x->k + x->m == KE;  // FP64 kernels: exact sizes
  const MulCtConst& mc = x->host_mc[lane];
  const MulCtConst* dmc = x->d_mc + lane;
  if (lift) {
    const LiftP<KQ, KE - KQ> P = make_lift_params<KQ, KE - KQ>(x, mc);
    const int64_t total = cnt << x->logn;  // cnt = polys
    if (compact) *compact = *compact && f64;  // only the FP64 lift writes the compact layout
    if (f64 && f64_product_period(x) == 12)
      lift_f64_kernel<KQ, KE - KQ, KQ + 2, 12><<<grid_for(total, 256), 256, 0, st>>>(
          in, out, cnt, x->logn, P, dmc, x->d_fallbacks, compact && *compact ? (lift_mode ? *lift_mode : 1) : 0);
    else if (f64)
      lift_f64_kernel<KQ, KE - KQ, KQ + 2><<<grid_for(total, 256), 256, 0, st>>>(
          in, out, cnt, x->logn, P, dmc, x->d_fallbacks, compact && *compact ? (lift_mode ? *lift_mode : 1) : 0);
    else
      lift_kernel<KQ, KE - KQ, KQ + 2><<<grid_for(total, 256), 256, 0, st>>>(in, out, cnt, x->logn, P, dmc,
                                                                             x->d_fallbacks);
    FCN_LAUNCH_CHECK(f64 ? "lift_f64_kernel" : "lift_kernel");
  } else {
    RescaleP<KQ, KE> P = make_rescale_params<KQ, KE>(x, mc);
    if (act && act->prescaled) {
      if (!f64) return set_error(FCN_ERR_STATE, "prescaled rescale inputs need the FP64 rescale kernel");
      P.prescaled = 1;
      P.dbl_in = act->dbl_in ? 1 : 0;
    }
    if (f64 && act && act->on) {
      P.act = 1;
      for (int i = 0; i < x->k; ++i) {
        const int64_t qi = (int64_t)x->primes[i];
        int64_t m2 = act->c2 % qi, m1 = act->c1 % qi;
        if (m2 < 0) m2 += qi;
        if (m1 < 0) m1 += qi;
        P.fc2[i] = h_signed((uint64_t)m2, (uint64_t)qi);
        P.fc2q[i] = P.fc2[i] / (double)qi;
        P.fc1[i] = h_signed((uint64_t)m1, (uint64_t)qi);
        P.fc1q[i] = P.fc1[i] / (double)qi;
      }
      act->applied = true;
    }
    const int64_t total = (cnt * 3) << x->logn;  // cnt = ciphertexts
    if (f64) {
      const int smem = 2 * (KE + KQ) * 256 * 8;
      int occ = 0;
      const void* fn = f64_product_period(x) == 12 ? (const void*)rescale_f64_kernel<KQ, KE, KQ + 2, 12>
                                                    : (const void*)rescale_f64_kernel<KQ, KE, KQ + 2>;
      FCN_CUDA(kernel_occupancy(fn, 256, smem, &occ));  // per-device smem attribute
      if (f64_product_period(x) == 12)
        rescale_f64_kernel<KQ, KE, KQ + 2, 12><<<grid_for(total, 256), 256, smem, st>>>(
            in, R01, DG, cnt, x->logn, P, dmc, x->d_fallbacks, act ? act->lin : nullptr);
      else
        rescale_f64_kernel<KQ, KE, KQ + 2><<<grid_for(total, 256), 256, smem, st>>>(
            in, R01, DG, cnt, x->logn, P, dmc, x->d_fallbacks, act ? act->lin : nullptr);
    }
    else
      rescale_kernel<KQ, KE, KQ + 2><<<grid_for(total, 256), 256, 0, st>>>(in, R01, DG, cnt, x->logn, P, dmc,
                                                                           x->d_fallbacks);
    FCN_LAUNCH_CHECK(f64 ? "rescale_f64_kernel" : "rescale_kernel");
  }
  return FCN_OK;
}

// The (KQ, KE) instantiation lift_or_rescale picks for a context, and
// whether its FP64 (exact-size) kernels run.
static bool f64_lift_rescale(const fcn_ctx* x) {
  // every k in 2..8 of 50-bit limbs (K = k + ceil((log2 n + 50.1 k + 4) / 50)) and cfg1's 37-bit (3, 6);
  // a single limb keeps the integer kernels
  static const int sizes[][2] = {{2, 5}, {2, 6}, {3, 6}, {3, 7}, {4, 8}, {4, 9}, {5, 11}, {6, 12},
                                 {6, 13}, {7, 15}, {8, 16}, {8, 17}, {16, 32}};
  for (const auto& sz : sizes)
    if (x->k <= sz[0] && x->m <= sz[1] - sz[0]) return x->fp && x->k == sz[0] && x->k + x->m == sz[1];
  return false;
}

static int lift_or_rescale(bool lift, const fcn_ctx* x, int lane, const uint64_t* in, uint64_t* out, int64_t cnt,
                           uint64_t* R01, uint64_t* DG, cudaStream_t st, ActArgs* act = nullptr,
                           bool* compact = nullptr, const int* lift_mode = nullptr) {
  const int k = x->k, m = x->m;
#define FCN_TRY(KQ, KE) \
  if (k <= KQ && m <= KE - KQ)                                                                                   \
    return run_lift_rescale<KQ, KE>(lift, x, lane, in, out, cnt, R01, DG, st, act, compact, lift_mode);
  FCN_TRY(2, 5)
  FCN_TRY(2, 6)
  FCN_TRY(3, 6)
  FCN_TRY(3, 7)
  FCN_TRY(4, 8)
  FCN_TRY(4, 9)
  FCN_TRY(5, 11)
  FCN_TRY(6, 12)
  FCN_TRY(6, 13)
  FCN_TRY(7, 15)
  FCN_TRY(8, 16)
  FCN_TRY(8, 17)
  FCN_TRY(16, 32)
#undef FCN_TRY
  return set_error(FCN_ERR_PARAM, "unsupported limb counts k=%d m=%d", k, m);
}

// Whether the square pipeline's workspace rows stay signed doubles between its
// FP64 kernels (FCN_DBL_ROWS=0: canonical u64 rows, A/B tests).  Needs the
// FP64 key MAC (at most 12 digits, keys converted) and the fused epilogue.
static bool dbl_rows(const fcn_ctx* x) {
  static const bool on = [] {
    const char* ev = getenv("FCN_DBL_ROWS");
    return !(ev && ev[0] == '0');
  }();
  return on && x->fp && x->ell + 1 <= 12;
}

// The q-limb inverse twist n^-1 psi_l^-j times (c2 mod q_l) as {w, w/q_l}
// (layout of fcn_ring::d_ftwist's first k limbs), cached per c2.  Returns
// nullptr when it would have to be built while the stream is being captured
// into a CUDA graph (no allocation there): the caller keeps the scaling
// epilogue.  FCN_TWIST_C2=0 disables it (A/B tests).
static const double2* c2_twist(fcn_ctx* x, int64_t c2, cudaStream_t st) {
  static const bool on = [] {
    const char* ev = getenv("FCN_TWIST_C2");
    return !(ev && ev[0] == '0');
  }();
  if (!on) return nullptr;
  std::lock_guard<std::mutex> lk(x->twist_mu);
  auto it = x->ftwist_c2.find(c2);
  if (it != x->ftwist_c2.end()) return it->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  const int k = x->k, n = x->n;
  std::vector<double2> tw((size_t)k * n);
  for (int l = 0; l < k; ++l) {
    const uint64_t q = x->primes[l];
    const int64_t m = c2 % (int64_t)q;
    const uint64_t cm = (uint64_t)(m < 0 ? m + (int64_t)q : m);
    const uint64_t iroot = h_powmod(x->ext->roots[l], q - 2, q);
    uint64_t w = h_mulmod(h_powmod((uint64_t)n % q, q - 2, q), cm, q);
    for (int j = 0; j < n; ++j) {
      const double ws = w > q / 2 ? -(double)(q - w) : (double)w;
      tw[(size_t)l * n + j] = make_double2(ws, ws / (double)q);
      w = h_mulmod(w, iroot, q);
    }
  }
  double2* d = nullptr;
  if (cudaMalloc(&d, sizeof(double2) * tw.size()) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  // ordered on the caller's stream and complete before the host table goes away
  if (cudaMemcpyAsync(d, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    cudaFree(d);
    cudaGetLastError();
    return nullptr;
  }
  x->ftwist_c2[c2] = d;
  return d;
}

// FCN_MAC_SGN=0: the MAC keeps separate positive / negative accumulators (A/B tests).
static bool mac_sgn_enabled() {
  static const bool on = [] {
    const char* ev = getenv("FCN_MAC_SGN");
    return !(ev && ev[0] == '0');
  }();
  return on;
}

// FCN_PRESCALE=0 keeps (B/b_j)^-1 in the rescale kernel instead of the INTT twist (A/B tests).
static bool prescale_enabled() {
  static const bool on = [] {
    const char* ev = getenv("FCN_PRESCALE");
    return !(ev && ev[0] == '0');
  }();
  return on;
}

// FCN_SQ_FUSE=0 disables the fused forward-NTT + tensor kernel (A/B tests).
static bool sq_fuse_enabled() {
  static const bool on = [] {
    const char* ev = getenv("FCN_SQ_FUSE");
    return !(ev && ev[0] == '0');
  }();
  return on;
}

static int launch_keymac(const uint64_t* DG, const fcn_keys* keys, uint64_t* ACC, int64_t C, int D, int k, const fcn_ctx* x,
                         cudaStream_t st, bool dbl = false) {
  const int64_t kn = (int64_t)k * x->n;  // one residue per thread
  const int bx = (int)((kn + 255) / 256);
  int64_t split = (148LL * 1024 * 4 + kn - 1) / kn;
  if (split > C) split = C;
  if (split < 1) split = 1;
  dim3 grid(bx, (unsigned)split);
  if (dbl && !(keys->d_fg && D <= 12)) return set_error(FCN_ERR_STATE, "double-format rows need the FP64 key MAC");
  if (keys->d_fg && D <= 12) {
    // exact digit count as the template argument: key words of unused digits take no registers;
    // beyond 8 digits only the key words stay in registers (LEAN); beyond 12 they spill: integer kernel
    switch (D) {
#define FCN_KM(DD, LN)                                                                                            \
  case DD:                                                                                                        \
    if (dbl)                                                                                                      \
      keymac_f64_kernel<DD, LN, true><<<grid, 256, 0, st>>>(DG, keys->d_fg, keys->d_fa, ACC, C, DD, k, x->logn,    \
                                                              x->ext->d_lc);                                      \
    else                                                                                                          \
      keymac_f64_kernel<DD, LN, false><<<grid, 256, 0, st>>>(DG, keys->d_fg, keys->d_fa, ACC, C, DD, k, x->logn,   \
                                                               x->ext->d_lc);                                     \
    break;
      FCN_KM(1, 1 >= FCN_KM_LEAN_FROM) FCN_KM(2, 2 >= FCN_KM_LEAN_FROM) FCN_KM(3, 3 >= FCN_KM_LEAN_FROM)
      FCN_KM(4, 4 >= FCN_KM_LEAN_FROM) FCN_KM(5, 5 >= FCN_KM_LEAN_FROM) FCN_KM(6, 6 >= FCN_KM_LEAN_FROM)
      FCN_KM(7, 7 >= FCN_KM_LEAN_FROM) FCN_KM(8, 8 >= FCN_KM_LEAN_FROM) FCN_KM(9, true) FCN_KM(10, true)
      FCN_KM(11, true) FCN_KM(12, true)
#undef FCN_KM
    }
    FCN_LAUNCH_CHECK("keymac_f64_kernel");
    return FCN_OK;
  }
  if (D <= 4)
    keymac_kernel<4><<<grid, 256, 0, st>>>(DG, keys->d_g, keys->d_a, ACC, C, D, k, x->logn, x->ext->d_lc);
  else if (D <= 8)
    keymac_kernel<8><<<grid, 256, 0, st>>>(DG, keys->d_g, keys->d_a, ACC, C, D, k, x->logn, x->ext->d_lc);
  else if (D <= 16)
    keymac_kernel<16><<<grid, 256, 0, st>>>(DG, keys->d_g, keys->d_a, ACC, C, D, k, x->logn, x->ext->d_lc);
  else
    keymac_kernel<32><<<grid, 256, 0, st>>>(DG, keys->d_g, keys->d_a, ACC, C, D, k, x->logn, x->ext->d_lc);
  FCN_LAUNCH_CHECK("keymac_kernel");
  return FCN_OK;
}

#ifndef FCN_KMP_LEAN_FROM
#define FCN_KMP_LEAN_FROM FCN_KM_LEAN_FROM
#endif
static int launch_keymac_pair(const uint64_t* DG, const fcn_keys* keys, uint64_t* ACCS, uint64_t* ACCP, int64_t C, int D,
                              int k, const fcn_ctx* x, cudaStream_t st) {
  const int64_t vn = (int64_t)(2 * k - 2) * x->n;  // one residue of one virtual limb per thread
  const int bx = (int)((vn + 255) / 256);
  int64_t split = (148LL * 1024 * 4 + vn - 1) / vn;
  if (split > C) split = C;
  if (split < 1) split = 1;
  dim3 grid(bx, (unsigned)split);
  switch (D) {
#define FCN_KMP(DD, LN)                                                                                              \
  case DD:                                                                                                           \
    keymac_pair_f64_kernel<DD, LN><<<grid, 256, 0, st>>>(DG, keys->d_pg, keys->d_pa, ACCS, ACCP, C, DD, k, x->logn, \
                                                         x->ext->d_lc);                                              \
    break;
    FCN_KMP(1, 1 >= FCN_KMP_LEAN_FROM) FCN_KMP(2, 2 >= FCN_KMP_LEAN_FROM) FCN_KMP(3, 3 >= FCN_KMP_LEAN_FROM)
    FCN_KMP(4, 4 >= FCN_KMP_LEAN_FROM) FCN_KMP(5, 5 >= FCN_KMP_LEAN_FROM) FCN_KMP(6, 6 >= FCN_KMP_LEAN_FROM)
    FCN_KMP(7, 7 >= FCN_KMP_LEAN_FROM) FCN_KMP(8, 8 >= FCN_KMP_LEAN_FROM) FCN_KMP(9, 9 >= FCN_KMP_LEAN_FROM)
    FCN_KMP(10, 10 >= FCN_KMP_LEAN_FROM) FCN_KMP(11, 11 >= FCN_KMP_LEAN_FROM) FCN_KMP(12, 12 >= FCN_KMP_LEAN_FROM)
#undef FCN_KMP
    default: return set_error(FCN_ERR_STATE, "shared-pair key MAC: %d digits", D);
  }
  FCN_LAUNCH_CHECK("keymac_pair_f64_kernel");
  return FCN_OK;
}

// ---- per-stage CUDA-event timing of fcn_mul_ct_multi (fcn_stage_timing):
// stage ids 0 lift, 1 forward NTT (+ fused tensor), 2 tensor INTT, 3 exact
// rescale + digits, 4 digit NTT, 5 key MAC, 6 final INTT + epilogue.
namespace {
struct StageTimer {
  std::mutex mu;
  bool on = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> recs;
};
StageTimer& stage_timer() {
  static StageTimer t;
  return t;
}
struct StageScope {
  cudaStream_t st;
  int id;
  cudaEvent_t e1 = nullptr;
  StageScope(int id_, cudaStream_t s) : st(s), id(id_) {
    StageTimer& T = stage_timer();
    if (!T.on) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    cudaEvent_t e0;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
      cudaGetLastError();
      e1 = nullptr;
      return;
    }
    cudaEventRecord(e0, st);
    std::lock_guard<std::mutex> lk(T.mu);
    T.recs.push_back({id, {e0, e1}});
  }
  ~StageScope() {
    if (e1) cudaEventRecord(e1, st);
  }
};
}  // namespace

extern "C" int fcn_stage_timing(int enable) {
  StageTimer& T = stage_timer();
  std::lock_guard<std::mutex> lk(T.mu);
  for (auto& r : T.recs) {
    cudaEventDestroy(r.second.first);
    cudaEventDestroy(r.second.second);
  }
  T.recs.clear();
  T.on = enable != 0;
  return FCN_OK;
}

extern "C" int fcn_stage_times(double* ms_out, int n_stages) {
  if (!ms_out || n_stages < 1) return set_error(FCN_ERR_ARG, "null output");
  for (int i = 0; i < n_stages; ++i) ms_out[i] = 0.0;
  StageTimer& T = stage_timer();
  std::lock_guard<std::mutex> lk(T.mu);
  for (auto& r : T.recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.second.second) != cudaSuccess ||
        cudaEventElapsedTime(&ms, r.second.first, r.second.second) != cudaSuccess)
      return set_error(FCN_ERR_CUDA, "stage event query failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (r.first >= 0 && r.first < n_stages) ms_out[r.first] += ms;
  }
  return FCN_OK;
}

extern "C" int fcn_mul_ct(const fcn_ctx* x, const fcn_keys* keys, int lane, const uint64_t* d_a, const uint64_t* d_b,
                          uint64_t* d_out, int64_t count, void* d_workspace, size_t workspace_bytes, void* stream) {
  return fcn_mul_ct_ex(x, keys, lane, d_a, d_b, d_out, count, 0, 1, 0, d_workspace, workspace_bytes, stream);
}

extern "C" int fcn_mul_ct_ex(const fcn_ctx* x, const fcn_keys* keys, int lane, const uint64_t* d_a, const uint64_t* d_b,
                             uint64_t* d_out, int64_t count, int flags, int64_t act_c2, int64_t act_c1, void* d_workspace,
                             size_t workspace_bytes, void* stream) {
  uint64_t* outs[1] = {d_out};
  return fcn_mul_ct_multi(x, keys, lane, d_a, d_b, outs, 1, count, flags, act_c2, act_c1, d_workspace, workspace_bytes,
                          stream);
}

extern "C" int fcn_mul_ct_multi(const fcn_ctx* x, const fcn_keys* keys, int lane, const uint64_t* d_a, const uint64_t* d_b,
                                uint64_t* const* d_outs, int n_dst, int64_t count, int flags, int64_t act_c2,
                                int64_t act_c1, void* d_workspace, size_t workspace_bytes, void* stream) {
  if (n_dst < 1 || n_dst > kMaxFanout || !d_outs) return set_error(FCN_ERR_ARG, "1..%d destinations", kMaxFanout);
  for (int d = 0; d < n_dst; ++d)
    if (!d_outs[d]) return set_error(FCN_ERR_ARG, "null destination %d", d);
  if (!x || !keys) return set_error(FCN_ERR_ARG, "null context or keys");
  if (lane < 0 || lane >= x->n_lanes) return set_error(FCN_ERR_ARG, "lane %d out of range", lane);
  if (count <= 0) return FCN_OK;
  if (x->ell + 1 > 32) return set_error(FCN_ERR_PARAM, "more than 32 decomposition digits");
  if (!d_a || !d_workspace) return set_error(FCN_ERR_ARG, "null buffer");
  if (keys->k != x->k || keys->n != x->n || keys->D != x->ell + 1) return set_error(FCN_ERR_ARG, "keys do not match context");
  const int64_t per = mulct_words_per_ct(x);
  const int64_t chunk_max = (int64_t)(workspace_bytes / 8) / per;
  if (chunk_max < 1) return set_error(FCN_ERR_STATE, "workspace too small (%zu bytes; need %lld per ciphertext)", workspace_bytes, (long long)(per * 8));
  DeviceGuard gd(x->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int k = x->k, K = x->k + x->m, D = x->ell + 1, n = x->n, logn = x->logn;
  const bool direct = x->host_mc[lane].direct != 0;
  const int64_t ct_words = 2LL * k * n;
  const bool act = (flags & FCN_MUL_ACT) != 0;
  if (act && d_b) return set_error(FCN_ERR_ARG, "the activation epilogue applies to squares only (b must be null)");
  NttEpi epi;
  for (int l = 0; l < k; ++l) {
    const uint64_t ql = x->primes[l];
    const int64_t m2 = act_c2 % (int64_t)ql, m1 = act_c1 % (int64_t)ql;
    epi.c2[l] = (uint64_t)(m2 < 0 ? m2 + (int64_t)ql : m2);
    epi.c1[l] = (uint64_t)(m1 < 0 ? m1 + (int64_t)ql : m1);
    epi.fc2[l] = h_signed(epi.c2[l], ql);
    epi.fc2q[l] = epi.fc2[l] / (double)ql;
    epi.fc1[l] = h_signed(epi.c1[l], ql);
    epi.fc1q[l] = epi.fc1[l] / (double)ql;
  }
  for (int64_t off = 0; off < count; off += chunk_max) {
    const int64_t C = (count - off) < chunk_max ? (count - off) : chunk_max;
    uint64_t* ws = (uint64_t*)d_workspace;
    uint64_t* EA = ws;
    uint64_t* EB = EA + C * 2 * K * n;
    uint64_t* T = EB + C * 2 * K * n;
    uint64_t* R01 = T + C * 3 * K * n;
    uint64_t* DGN = R01 + C * 2 * k * n;
    uint64_t* ACC = DGN + C * D * k * n;
    uint64_t* DGR = ACC + C * 2 * k * n;
    const uint64_t* a = d_a + off * ct_words;
    const uint64_t* b = d_b ? d_b + off * ct_words : nullptr;
    // (i) lift + forward NTT over the extended base, (ii) tensor.  Squares on
    // FP64 rings: compact lift (auxiliary rows only) and one fused
    // forward-NTT + tensor kernel that reads the q-limb rows from a itself.
    bool fused = !b && x->fp && sq_fuse_enabled() && logn >= 10 && logn <= 14;
    // the tensor INTT's twist also applies the rescale's first factor
    // (B/b_j)^-1 on the FP64 path (one multiply per residue saved), and the
    // square pipeline keeps its workspace rows as signed doubles from the
    // compact lift to the final INTT (no u64 round trips in between)
    const bool prescale = x->d_ftwist_binv && ntt_family(x->ext, K, 0) == 2 && f64_lift_rescale(x) && prescale_enabled();
    const bool want_dbl = fused && prescale && dbl_rows(x);
    if (fused) {
      int lift_mode = want_dbl ? 2 : 1;  // compact lift; 2: auxiliary rows as signed doubles
      int rc;
      {
        StageScope ss(0, st);
        rc = lift_or_rescale(true, x, lane, a, EA, C * 2, nullptr, nullptr, st, nullptr, &fused, &lift_mode);
      }
      if (rc) return rc;
      StageScope ss(1, st);
      if (fused) {
        rc = launch_ntt_square_tensor(x->ext, a, EA, T, C, k, x->m, st, want_dbl);
        if (rc) return rc < 0 ? rc : set_error(FCN_ERR_STATE, "fused square tensor unavailable");
      } else {  // the lift wrote the full extended rows
        rc = launch_ntt(x->ext, EA, C * 2 * K, K, 0, true, st);
        if (rc) return rc;
      }
    } else {
      for (int which = 0; which < (b ? 2 : 1); ++which) {
        uint64_t* dst = which ? EB : EA;
        int rc;
        {
          StageScope ss(0, st);
          rc = lift_or_rescale(true, x, lane, which ? b : a, dst, C * 2, nullptr, nullptr, st);
        }
        if (rc) return rc;
        StageScope ss(1, st);
        rc = launch_ntt(x->ext, dst, C * 2 * K, K, 0, true, st);
        if (rc) return rc;
      }
    }
    if (!fused) {
      StageScope ss(1, st);
      if (x->fp)
        tensor_f64_kernel<<<grid_for((C * K) << (logn - 1), 256), 256, 0, st>>>(EA, b ? EB : nullptr, T, C, K, logn,
                                                                                x->ext->d_lc);
      else
        tensor_kernel<<<grid_for((C * K) << (logn - 1), 256), 256, 0, st>>>(EA, b ? EB : nullptr, T, C, K, logn,
                                                                            x->ext->d_lc);
      FCN_LAUNCH_CHECK(x->fp ? "tensor_f64_kernel" : "tensor_kernel");
    }
    // (iii) inverse NTT
    const bool dbl = fused && want_dbl;
    NttEpi tw_epi;
    tw_epi.mode = 0;
    tw_epi.ftwist = x->d_ftwist_binv;
    tw_epi.dbl = dbl;
    int rc;
    {
      StageScope ss(2, st);
      rc = launch_ntt(x->ext, T, C * 3 * K, K, 0, false, st, nullptr, 1, prescale ? &tw_epi : nullptr);
    }
    if (rc) return rc;
    // (iv) exact rescale + digit decomposition (FP64: R01 <- c2 R01 + c1 a for the activation)
    ActArgs aa;
    aa.on = act;
    aa.c2 = act_c2;
    aa.c1 = act_c1;
    aa.lin = a;
    aa.prescaled = prescale;
    aa.dbl_in = dbl;
    {
      StageScope ss(3, st);
      rc = lift_or_rescale(false, x, lane, T, nullptr, C, R01, direct ? DGR : DGN, st, &aa);
    }
    if (rc) return rc;
    epi.mode = !act ? 1 : (aa.applied ? 3 : 2);
    epi.ftwist = nullptr;
    if (epi.mode == 3 && x->fp && ntt_family(x->ext, k, 0) == 2) {
      // out = R + c2 INTT(ACC) == R + INTT'(ACC) with c2 folded into the twist
      if (const double2* tw = c2_twist(const_cast<fcn_ctx*>(x), act_c2, st)) {
        epi.mode = 1;
        epi.ftwist = tw;
      }
    }
    // (v) digits to NTT (broadcast rows when digits are limb-independent), key MAC
    NttEpi dg_epi;
    dg_epi.dbl = dbl;
    if (x->pair && dbl && direct && keys->d_pg && (epi.mode == 1 || epi.mode == 3)) {
      // shared-pair relinearisation: digits under q_0, q_1 only (2D rows per
      // ciphertext instead of D k); limbs 0, 1 finish as usual, limbs j >= 2
      // through the two-residue CRT of ntt_f64_inv_pair.  The 2D digit rows
      // and the 4k - 4 accumulator rows share the D k + 2k rows of DGN | ACC.
      uint64_t* ACCS = DGN + C * 2 * D * n;
      uint64_t* ACCP = ACCS + C * 4 * n;
      {
        StageScope ss(4, st);
        rc = launch_ntt(x->ext, DGN, C * D * 2, 2, 0, true, st, DGR, 2, &dg_epi);
      }
      if (rc) return rc;
      {
        StageScope ss(5, st);
        rc = launch_keymac_pair(DGN, keys, ACCS, ACCP, C, D, k, x, st);
      }
      if (rc) return rc;
      StageScope ss(6, st);
      epi.add = R01;
      epi.lin = a;
      epi.dbl = dbl;
      epi.in_per = 2;
      epi.out_per = k;
      epi.out.n = n_dst;
      for (int d = 0; d < n_dst; ++d) epi.out.dst[d] = d_outs[d] + off * ct_words;
      rc = launch_ntt(x->ext, ACCS, C * 4, 2, 0, false, st, nullptr, 1, &epi);
      if (rc) return rc;
      PairEpi pe;
      pe.add = R01;
      pe.out = epi.out;
      pe.kq = k;
      pe.inv01 = x->pair_inv01;
      pe.inv01q = x->pair_inv01q;
      const bool scale = epi.mode == 3 || epi.ftwist != nullptr;  // c2 (folded into the single rows' twist or not)
      for (int l = 0; l < k; ++l) {
        pe.c0[l] = x->pair_c0[l];
        pe.c0q[l] = x->pair_c0q[l];
        pe.fc2[l] = epi.fc2[l];
        pe.fc2q[l] = epi.fc2q[l];
      }
      rc = launch_ntt_pair(x->ext, ACCP, C * 2 * (k - 2), scale, st, &pe);
      if (rc) return rc;
      continue;
    }
    {
      StageScope ss(4, st);
      if (direct)
        rc = launch_ntt(x->ext, DGN, C * D * k, k, 0, true, st, DGR, k, dbl ? &dg_epi : nullptr);
      else
        rc = launch_ntt(x->ext, DGN, C * D * k, k, 0, true, st, nullptr, 1, dbl ? &dg_epi : nullptr);
    }
    if (rc) return rc;
    {
      StageScope ss(5, st);
      rc = launch_keymac(DGN, keys, ACC, C, D, k, x, st, dbl);
    }
    if (rc) return rc;
    // (vi) inverse NTT with the fused epilogue: out = R01 + INTT(ACC)
    //      [ * c2 + c1 * a  when FCN_MUL_ACT: the a2 x^2 + a1 x activation]
    epi.add = R01;
    epi.lin = a;
    epi.dbl = dbl;
    epi.out.n = n_dst;
    for (int d = 0; d < n_dst; ++d) epi.out.dst[d] = d_outs[d] + off * ct_words;
    {
      StageScope ss(6, st);
      rc = launch_ntt(x->ext, ACC, C * 2 * k, k, 0, false, st, nullptr, 1, &epi);
    }
    if (rc) return rc;
  }
  return FCN_OK;
}

extern "C" int fcn_key_mac(const fcn_ctx* x, const fcn_keys* keys, const uint64_t* d_digits, uint64_t* d_acc,
                           int64_t count, void* stream) {
  if (!x || !keys) return set_error(FCN_ERR_ARG, "null context or keys");
  if (count <= 0) return FCN_OK;
  if (!d_digits || !d_acc) return set_error(FCN_ERR_ARG, "null buffer");
  if (keys->k != x->k || keys->n != x->n || keys->D != x->ell + 1) return set_error(FCN_ERR_ARG, "keys do not match context");
  DeviceGuard gd(x->device);
  return launch_keymac(d_digits, keys, d_acc, count, keys->D, x->k, x, (cudaStream_t)stream);
}

extern "C" int fcn_noise_max(const fcn_ctx* x, int lane, const uint64_t* d_w, int64_t count, uint64_t* d_out,
                             int blocks, int out_words, void* stream) {
  if (!x || lane < 0 || lane >= x->n_lanes) return set_error(FCN_ERR_ARG, "bad context or lane");
  if (count <= 0) return FCN_OK;
  if (!d_w || !d_out || blocks < 1 || count > 65535) return set_error(FCN_ERR_ARG, "bad buffers or sizes");
  const int qwords = x->host_mc[lane].qwords;
  if (out_words < qwords || out_words > 256) return set_error(FCN_ERR_ARG, "out_words must be >= %d", qwords);
  DeviceGuard g(x->device);
  cudaStream_t st = (cudaStream_t)stream;
  const MulCtConst* mc = x->d_mc + lane;
  dim3 grid((unsigned)blocks, (unsigned)count);
  if (x->k <= 4)
    noise_max_kernel<4, 6><<<grid, 256, 0, st>>>(d_w, x->logn, mc, x->ext->d_lc, d_out, out_words);
  else if (x->k <= 8)
    noise_max_kernel<8, 10><<<grid, 256, 0, st>>>(d_w, x->logn, mc, x->ext->d_lc, d_out, out_words);
  else
    noise_max_kernel<16, 18><<<grid, 256, 0, st>>>(d_w, x->logn, mc, x->ext->d_lc, d_out, out_words);
  FCN_LAUNCH_CHECK("noise_max_kernel");
  return FCN_OK;
}

extern "C" int fcn_decrypt_round(const fcn_ctx* x, int lane, const uint64_t* d_w, uint64_t* d_m, int64_t count, void* stream) {
  if (!x || lane < 0 || lane >= x->n_lanes) return set_error(FCN_ERR_ARG, "bad context or lane");
  if (count <= 0) return FCN_OK;
  if (!d_w || !d_m) return set_error(FCN_ERR_ARG, "null buffer");
  DeviceGuard g(x->device);
  const int64_t total = count << x->logn;
  cudaStream_t st = (cudaStream_t)stream;
  const MulCtConst* mc = x->d_mc + lane;
  if (x->k <= 4)
    decrypt_round_kernel<4, 6><<<grid_for(total, 256), 256, 0, st>>>(d_w, d_m, count, x->logn, mc, x->ext->d_lc, x->d_fallbacks);
  else if (x->k <= 8)
    decrypt_round_kernel<8, 10><<<grid_for(total, 256), 256, 0, st>>>(d_w, d_m, count, x->logn, mc, x->ext->d_lc, x->d_fallbacks);
  else
    decrypt_round_kernel<16, 18><<<grid_for(total, 256), 256, 0, st>>>(d_w, d_m, count, x->logn, mc, x->ext->d_lc, x->d_fallbacks);
  FCN_LAUNCH_CHECK("decrypt_round_kernel");
  return FCN_OK;
}
