// Internal definitions shared by the libfcn translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/fcn.h"

namespace fcn {

// ------------------------------------------------------------------ errors

int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
#define FCN_CUDA(call)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return check_cuda(_e, #call); \
  } while (0)
extern std::atomic<long long> g_launches;  // kernels launched by this library
#define FCN_LAUNCH_CHECK(what)                                 \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return check_cuda(_e, what);        \
    ::fcn::g_launches.fetch_add(1, std::memory_order_relaxed); \
  } while (0)

// Per-device kernel setup (dynamic shared-memory attribute + resident CTAs
// per SM), cached per (kernel, device, smem) under a lock: the attribute is a
// per-device property, so one process driving several devices sets it on
// each (csrc/ring.cu).  Returns the CUDA error of the setup.
cudaError_t kernel_occupancy(const void* fn, int threads, size_t smem, int* occ_out);
// SM count of the current device (cached per device).
int device_sms();

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------ limb tables

// Per-limb constants, one struct per prime of a ring (device resident).
struct LimbConst {
  uint64_t q;       // the prime, < 2^62
  uint64_t q2;      // 2q
  uint64_t ninv;    // n^-1 mod q
  uint64_t ninv_s;  // Shoup quotient floor(ninv 2^64 / q)
  uint64_t wlast;   // ipsi[1] * n^-1 mod q (last inverse stage, merged scaling)
  uint64_t wlast_s;
  uint64_t mu;      // Barrett floor(2^(2s) / q), s = bitlen(q)
  uint32_t s;       // bitlen(q)
  uint32_t pad;
  uint64_t one_s;   // floor(2^64 / q): Shoup quotient of the constant 1
  uint64_t r64;     // 2^64 mod q
  uint64_t r64_s;
  uint64_t nq;      // 2^64 - q
  uint32_t m32;     // floor(2^64 / q) when q > 2^32, else 0
  uint32_t pad2;
  double fq;        // q as a double (exact), for the FP64 path (q < 2^51)
  double fqi;       // 1 / q rounded
};

struct __align__(16) Twiddle {
  uint64_t w;  // psi^bitrev(i) (forward) or psi^-bitrev(i) (inverse)
  uint64_t s;  // floor(w 2^64 / q)
};

}  // namespace fcn

struct fcn_ring {
  int device = 0;
  int n = 0;
  int logn = 0;
  int L = 0;
  std::vector<uint64_t> primes;
  std::vector<uint64_t> roots;
  std::vector<fcn::LimbConst> host_lc;
  fcn::LimbConst* d_lc = nullptr;  // [L]
  fcn::Twiddle* d_fwd = nullptr;   // [L][n]
  fcn::Twiddle* d_inv = nullptr;   // [L][n]
  fcn::Twiddle* d_ict = nullptr;   // [L][n] DIT inverse twiddles: [2^s + k] = psi^-(k n / 2^s)
  fcn::Twiddle* d_twist = nullptr; // [L][n] n^-1 psi^-j
  // forward twiddles of the last five stages laid out for coalesced loads in
  // the register pass that owns 32 contiguous residues per thread:
  // [L][u][blk][t] = psi[2^(logn-5+u) + t 2^u + blk], t < n/32 (n >= 32)
  fcn::Twiddle* d_fwd_last = nullptr;
  // FP64 copies of the four NTT tables for limbs below 2^51 (fp_ok): each
  // entry {w, w / q} with w the signed representative in (-q/2, q/2].
  bool fp_ok = false;
  double2* d_ffwd = nullptr;
  double2* d_fict = nullptr;
  double2* d_ftwist = nullptr;
  double2* d_ffl = nullptr;
};

namespace fcn {

// ------------------------------------------------------ device arithmetic

__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t m) { return x >= m ? x - m : x; }

// a * w mod q in [0, 2q) for constant w < q with ws = floor(w 2^64 / q); any a < 2^64.
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
  return a * w - __umul64hi(a, ws) * q;
}
__device__ __forceinline__ uint64_t shoup(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
  return csub(shoup_lazy(a, w, ws, q), q);
}
// Exact (quotient, remainder) of a * w / q for constant w with Shoup quotient ws.
__device__ __forceinline__ uint64_t shoup_divmod(uint64_t a, uint64_t w, uint64_t ws, uint64_t q,
                                                 uint64_t* quo) {
  uint64_t h = __umul64hi(a, ws);
  uint64_t r = a * w - h * q;
  if (r >= q) {
    r -= q;
    h += 1;
  }
  *quo = h;
  return r;
}

// Barrett: (hi:lo) mod q for a 128-bit x < q^2 (q < 2^62).  Canonical.
__device__ __forceinline__ uint64_t barrett128(uint64_t hi, uint64_t lo, const LimbConst& c) {
  const uint32_t s = c.s;
  // x1 = x >> (s - 1) fits in s + 1 <= 63 bits
  uint64_t x1 = (lo >> (s - 1)) | (s - 1 == 0 ? 0 : (hi << (65 - s)));
  // qhat = (x1 * mu) >> (s + 1)
  uint64_t ph = __umul64hi(x1, c.mu);
  uint64_t pl = x1 * c.mu;
  uint64_t qhat = (pl >> (s + 1)) | (ph << (63 - s));
  uint64_t r = lo - qhat * c.q;
  r = csub(r, c.q);
  return csub(r, c.q);
}

__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, const LimbConst& c) {
  return barrett128(__umul64hi(a, b), a * b, c);
}

// Any 128-bit (hi:lo) mod q, canonical: hi*2^64 + lo folded through Shoup.
__device__ __forceinline__ uint64_t reduce128(uint64_t hi, uint64_t lo, const LimbConst& c) {
  uint64_t a = csub(shoup_lazy(hi, c.r64, c.r64_s, c.q), c.q);
  uint64_t b = csub(shoup_lazy(lo, 1, c.one_s, c.q), c.q);
  return csub(a + b, c.q);
}

__device__ __forceinline__ void add128(uint64_t& hi, uint64_t& lo, uint64_t ph, uint64_t pl) {
  lo += pl;
  hi += ph + (lo < pl);
}

__device__ __forceinline__ uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
__device__ __forceinline__ uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + q - b, q); }

// a*w mod q in [0, 4q) for any a < 2^64, constant w < q with ws = floor(w 2^64/q),
// nq = 2^64 - q.  The quotient estimate h = a1 s1 + hi(a1 s0) + hi(a0 s1) omits
// a0*s0 and the low halves of the cross products, so it undershoots
// floor(a ws / 2^64) by at most 2 (remainder < 2q + 2q).  9 IMAD-pipe ops.
__device__ __forceinline__ uint64_t mulw(uint64_t a, uint64_t w, uint64_t ws, uint64_t nq) {
  uint64_t r;
  asm("{\n\t"
      ".reg .u32 a0, a1, w0, w1, s0, s1, n0, n1, hl, hh, rl, rh;\n\t"
      ".reg .u64 H, R;\n\t"
      "mov.b64 {a0, a1}, %1;\n\t"
      "mov.b64 {w0, w1}, %2;\n\t"
      "mov.b64 {s0, s1}, %3;\n\t"
      "mov.b64 {n0, n1}, %4;\n\t"
      "mul.wide.u32 H, a1, s1;\n\t"
      "mov.b64 {hl, hh}, H;\n\t"
      "mad.hi.cc.u32 hl, a1, s0, hl;\n\t"
      "addc.u32 hh, hh, 0;\n\t"
      "mad.hi.cc.u32 hl, a0, s1, hl;\n\t"
      "addc.u32 hh, hh, 0;\n\t"
      "mul.wide.u32 R, a0, w0;\n\t"
      "mad.wide.u32 R, hl, n0, R;\n\t"
      "mov.b64 {rl, rh}, R;\n\t"
      "mad.lo.u32 rh, a0, w1, rh;\n\t"
      "mad.lo.u32 rh, a1, w0, rh;\n\t"
      "mad.lo.u32 rh, hl, n1, rh;\n\t"
      "mad.lo.u32 rh, hh, n0, rh;\n\t"
      "mov.b64 %0, {rl, rh};\n\t"
      "}"
      : "=l"(r)
      : "l"(a), "l"(w), "l"(ws), "l"(nq));
  return r;
}

// x mod q for x < 2^62, 2^34 <= q < 2^56: quotient from the high word
// (m32 = floor(2^64/q)) undershoots by at most 1.
__device__ __forceinline__ uint64_t reduce_small(uint64_t x, uint32_t m32, uint64_t q) {
  const uint32_t qe = __umulhi((uint32_t)(x >> 32), m32);
  const uint64_t r = x - (uint64_t)qe * q;
  return r >= q ? r - q : r;
}

// async global -> shared copies (Ampere+ cp.async; completion per thread)
__device__ __forceinline__ void cp_async8(uint64_t* smem_dst, const uint64_t* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc));
}
// The same copy ordered after the value `dep` is available: the copy
// overwrites the shared-memory word `dep` was just read from, and naming it
// as an operand keeps the compiler from scheduling the copy above that read.
__device__ __forceinline__ void cp_async8_after(uint64_t* smem_dst, const uint64_t* gsrc, double dep) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;  // after %2\n" ::"r"(sa), "l"(gsrc), "d"(dep));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ----------------------------------------------- FP64 signed residues
// For q < 2^51 a residue is held as an integer-valued double x, |x| < 2^53
// (so every value and every intermediate below is exact).  The FP64 pipe
// issues these at ~60 ops/clk/SM on B200 (tools/fp64bench.cu), more than
// twice the integer mulw rate.

// r == a w (mod q), |r| < 1.5 q, for |a| < 2^53, |w| <= q/2, wq = RN(w/q):
// h + l = a w exactly (FMA error-free product); qt = rint(a wq) is within
// 1.5 of a w / q, so h - qt q and then + l are exact integers below 2^53.
__device__ __forceinline__ double fmulq(double a, double w, double wq, double q) {
  const double h = a * w;
  const double l = fma(a, w, -h);
  const double qt = rint(a * wq);
  return fma(-qt, q, h) + l;
}
// fmulq with the quotient rounded by the 1.5*2^52 magic constant (two FP64
// pipe ops instead of DMUL + FRND on the XU pipe); requires |a wq| < 2^51.
__device__ __forceinline__ double fmulq_m(double a, double w, double wq, double q) {
  const double M = 6755399441055744.0;
  const double h = a * w;
  const double l = fma(a, w, -h);
  const double qt = fma(a, wq, M) - M;
  return fma(-qt, q, h) + l;
}
// a b mod q for |a|, |b| <= q/2 + small (q < 2^51): |a b / q| < 2^49, so the
// magic-constant quotient is exact to 1/2 and the result is |.| < 0.6 q.
__device__ __forceinline__ double fprod(double a, double b, double q, double qi) {
  const double M = 6755399441055744.0;
  const double h = a * b;
  const double l = fma(a, b, -h);
  const double qt = fma(h, qi, M) - M;
  return fma(-qt, q, h) + l;
}
// x mod q centred: |r| <= q/2 + 2^-40 q for |x| < 2^53 and |x / q| < 2^10
// (every use: sums of a few reduced products or butterfly outputs).
// The quotient is rounded with the 1.5 * 2^52 magic constant (DFMA + DADD +
// DFMA); FCN_FRED_FRND=1 uses FRND instead (XU pipe, DMUL + FRND + DFMA), one
// FP64 operation fewer but measured slower: the NTT butterflies already keep
// the XU busy with their own FRND (kbench 0.370 -> 0.378 ms forward).  Either
// quotient is within 1/2 + |x/q| 2^-52 of x/q.
#ifndef FCN_FRED_FRND
#define FCN_FRED_FRND 0
#endif
__device__ __forceinline__ double fredq(double x, double qi, double q) {
#if FCN_FRED_FRND
  const double qt = rint(x * qi);
#else
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  const double qt = fma(x, qi, M) - M;
#endif
  return fma(-qt, q, x);
}
// Reduction schedules of the FP64 NTT (ntt_f64.cuh): reduce every value
// before stage s?  RS 0: s = 3, 6, 9, 12 (any q < 2^51); RS 1: once, before
// stage logn/2; RS 2: never.  ntt.cu f64_schedule checks the bound.
__host__ __device__ constexpr bool f64_red_before(int logn, int rs, int s) {
  return rs == 0 ? (s > 0 && s % 3 == 0) : rs == 1 ? (s == logn / 2) : false;
}
// u64 residue (< 2^52) <-> double, bit tricks instead of the slow I2F/F2I.
__device__ __forceinline__ double u2f(uint64_t x) {
  return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 4503599627370496.0;
}
// centred |x| <= q/2 + small (any |x| < q) -> canonical [0, q)
__device__ __forceinline__ uint64_t f2u_canon(double x, double q) {
  const double y = x < 0.0 ? x + q : x;
  return (uint64_t)__double_as_longlong(y + 4503599627370496.0) & 0x000FFFFFFFFFFFFFull;
}

// ---------------------------------------------------- host-side helpers

inline uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t m) {
  return (uint64_t)(((unsigned __int128)a * b) % m);
}
inline uint64_t h_powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = h_mulmod(r, b, m);
    b = h_mulmod(b, b, m);
    e >>= 1;
  }
  return r;
}
inline uint64_t h_shoup(uint64_t w, uint64_t q) { return (uint64_t)(((unsigned __int128)w << 64) / q); }
bool h_is_prime(uint64_t v);
int bitlen64(uint64_t v);
LimbConst make_limb_const(uint64_t q, int n, uint64_t ipsi1);
// Output fan-out: the final store of a kernel goes to every destination
// (this GPU's buffer and, for sharded evaluation, the peers' buffers mapped
// over NVLink), replacing the all-gather that would otherwise follow.
constexpr int kMaxFanout = 8;
struct Fanout {
  int n = 0;
  uint64_t* dst[kMaxFanout] = {};
};
// Tensor-core linear layer (csrc/mac_tc.cu): one output group = up to 128
// output rows (rows[row_off .. row_off + m)) over the inputs
// kidx[k_off .. k_off + n_k); its weights are nchunks = ceil(n_k / 64)
// pre-laid-out 8 KB K-major tiles starting at tile w_off of wimg.
struct TcGroup {
  int32_t row_off, m, k_off, n_k, w_off, pad0, pad1, pad2;
};
struct TcLaunch {
  const uint8_t* planes = nullptr;  // [n_in][P][cols] byte planes
  int64_t cols = 0;                 // residues per ciphertext (2 k n)
  int planes_n = 0;                 // P
  int64_t n_groups = 0;
  const TcGroup* groups = nullptr;
  const int32_t* kidx = nullptr;
  const int32_t* rows = nullptr;
  const int8_t* wimg = nullptr;
  Fanout out;                        // rows [row_lo, row_hi) of the layer's output
  int64_t row_lo = 0, row_hi = 0;
  int logn = 0, k = 0;
  const LimbConst* lcs = nullptr;
};
int launch_mac_tc(const TcLaunch& a, cudaStream_t st);
// Row pitch (bytes) of one byte plane of one ciphertext: the 2kn columns
// padded by 256 bytes, so the 64-byte segments the MAC gathers from
// thousands of planes do not all fall on the same L2 sets (2kn is a power
// of two times k).
__host__ __device__ inline int64_t tc_plane_pitch(int64_t cols) { return cols + 256; }
int launch_split_planes(const uint64_t* in, int64_t rows, int64_t cols, int P, uint8_t* planes, cudaStream_t st);

// Inverse-NTT epilogue (row-aligned with the transformed rows, period/offset
// limb indexing): mode 1: out = v + add; mode 2: out = c2 (v + add) + c1 lin;
// mode 3: out = add + c2 v (mod q_l).  Coefficients per limb index: canonical u64 and FP64 {w, w/q}.
constexpr int kEpiLimbs = 64;
struct NttEpi {
  int mode = 0;
  const uint64_t* add = nullptr;
  const uint64_t* lin = nullptr;
  Fanout out;  // destinations, row-aligned
  // mode 0 on the FP64 inverse: replacement twist table (n^-1 psi^-j times a
  // per-limb constant), e.g. the rescale's (B/b_l)^-1 folded into the tensor's INTT
  const double2* ftwist = nullptr;
  // FP64 kernels only: rows as signed residues in raw doubles instead of
  // canonical u64 (forward: output; plain inverse: input and output; epilogue
  // inverse: input), the internal format of the square pipeline
  int dbl = 0;
  uint64_t c2[kEpiLimbs], c1[kEpiLimbs];
  double fc2[kEpiLimbs], fc2q[kEpiLimbs], fc1[kEpiLimbs], fc1q[kEpiLimbs];
  // FP64 epilogue inverse only: input row r belongs to output row
  // (r / in_per) * out_per + r % in_per of add / out (0: the same row).  The
  // shared-pair relinearisation transforms only limbs 0 and 1 of every poly
  // this way (in_per = 2, out_per = k).
  int in_per = 0, out_per = 0;
};

// Shared-pair relinearisation (fv.cu): for a limb j >= 2 the
// key-switching sum V_j = sum_d lift(key_d mod q_j) * D_d is computed as an
// exact integer through its residues modulo the first two limbs q_0, q_1
// (|V_j| < q_0 q_1 / 2), so the digits are transformed under two primes
// instead of k.  ntt_f64_inv_pair inverts the two residue rows of one unit
// (ct, poly, j), rebuilds V_j = y0 + q_0 ((y1 - y0) q_0^-1 mod q_1) and writes
// out = add + c2 V_j (mod q_j).
constexpr int kPairLimbs = 16;
struct PairEpi {
  const uint64_t* add = nullptr;  // [C][2][k][n] signed doubles (R0 / R1)
  Fanout out;                     // [C][2][k][n] canonical u64
  int kq = 0;                     // limbs per poly (units per poly = kq - 2)
  double inv01 = 0, inv01q = 0;   // q_0^-1 mod q_1 (signed), / q_1
  double c0[kPairLimbs], c0q[kPairLimbs];    // q_0 mod q_j (signed), / q_j
  double fc2[kPairLimbs], fc2q[kPairLimbs];  // c2 mod q_j (signed), / q_j
};
// Inverse NTT of `units` row pairs [unit][2][n] (signed doubles, residues
// modulo limb 0 and limb 1 of ring r) with the CRT epilogue above; scale:
// multiply by c2.  FP64 rings with 2^10 <= n <= 2^14 only.
int launch_ntt_pair(const fcn_ring* r, uint64_t* d, int64_t units, bool scale, cudaStream_t st, const PairEpi* epi);
// Batched NTT over rows; the forward may read row r's input from
// src + (r / src_div) * n (broadcast of one source row to several limbs).
int launch_ntt(const fcn_ring* r, uint64_t* d, int64_t n_rows, int period, int offset, bool fwd, cudaStream_t st,
               const uint64_t* src = nullptr, int src_div = 1, const NttEpi* epi = nullptr);
// Which NTT kernels launch_ntt runs for rows of limbs offset .. offset+period-1:
// 0 generic (ntt_v1), 1 integer register passes (ntt_v2), 2 FP64 (ntt_f64.cuh).
int ntt_family(const fcn_ring* r, int period, int offset);
// Forward NTT of squared ciphertexts' lifted polys fused with the NTT-domain
// tensor (ntt_f64.cuh ntt_f64_fwd_sq): FP64 rings with 2^10 <= n <= 2^14 only
// (returns 1 when not applicable, nothing launched).
int launch_ntt_square_tensor(const fcn_ring* r, const uint64_t* a, const uint64_t* aux, uint64_t* Tout, int64_t C,
                             int k, int m, cudaStream_t st, bool dbl = false);

inline int grid_for(int64_t work, int block, int max_blocks = 148 * 16) {
  int64_t g = (work + block - 1) / block;
  if (g > max_blocks) g = max_blocks;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace fcn
