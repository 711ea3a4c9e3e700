// libfcn: RNS ring Z_q[x]/(x^n+1) on B200 -- tables, batched NTT, elementwise ops.
//
// Replaces reference ring.py (tables :67-101, transforms :199-255, elementwise
// :261-300, monomial :339-361) and modmath.py (:31-85).  Every kernel works on
// rows of n uint64 residues; a row's limb is (limb_offset + row % limb_period),
// so one launch covers a whole batch of ciphertexts [B][2][k][n].
//
// NTT design: one CTA per row (or per independent segment
// of a row when n > 16384).  The row is staged once in shared memory
// (padded by one word per 32 to keep strided group accesses conflict-light);
// butterflies run in registers on groups of 2^R elements spanning R stages
// (R <= 5), so a 14-stage transform is 3 smem round trips.  Twiddle factors
// are (w, floor(w 2^64/q)) pairs; the multiply is Shoup's with Harvey's lazy
// ranges ([0,4q) forward, [0,2q) inverse) and one canonicalisation at the
// end, so outputs are bit-identical to the reference's canonical-per-stage
// numpy transform.

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "fcn_common.cuh"

namespace fcn {

static thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  return set_error(FCN_ERR_CUDA, "CUDA error in %s: %s", what, cudaGetErrorString(e));
}

bool h_is_prime(uint64_t v) {
  static const uint64_t W[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (v < 2) return false;
  for (uint64_t w : W)
    if (v % w == 0) return v == w;
  uint64_t d = v - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++r;
  }
  for (uint64_t a : W) {
    uint64_t x = h_powmod(a, d, v);
    if (x == 1 || x == v - 1) continue;
    bool comp = true;
    for (int i = 0; i < r - 1; ++i) {
      x = h_mulmod(x, x, v);
      if (x == v - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}

int bitlen64(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

LimbConst make_limb_const(uint64_t q, int n, uint64_t ipsi1) {
  LimbConst c;
  memset(&c, 0, sizeof(c));
  c.q = q;
  c.q2 = 2 * q;
  c.ninv = h_powmod((uint64_t)n % q, q - 2, q);
  c.ninv_s = h_shoup(c.ninv, q);
  c.wlast = h_mulmod(ipsi1, c.ninv, q);
  c.wlast_s = h_shoup(c.wlast, q);
  c.s = (uint32_t)bitlen64(q);
  c.mu = (uint64_t)(((unsigned __int128)1 << (2 * c.s)) / q);
  c.one_s = h_shoup(1, q);
  c.r64 = (uint64_t)(((unsigned __int128)1 << 64) % q);
  c.r64_s = h_shoup(c.r64, q);
  return c;
}

// primitive_2n_root (modmath.py:136-149): smallest g in [2, 4096) whose
// g^((q-1)/2n) has order exactly 2n.
static bool root_2n(uint64_t q, int n, uint64_t* out) {
  if ((q - 1) % (2 * (uint64_t)n)) return false;
  uint64_t e = (q - 1) / (2 * (uint64_t)n);
  for (uint64_t g = 2; g < 4096; ++g) {
    uint64_t r = h_powmod(g, e, q);
    if (h_powmod(r, n, q) == q - 1) {
      *out = r;
      return true;
    }
  }
  return false;
}

static uint32_t bitrev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}

// ------------------------------------------------------------ NTT kernels

__device__ __forceinline__ int phys(int i) { return i + (i >> 5); }

// Forward CT pass over R stages (local stages ls0 .. ls0+R-1 of a segment of
// size S = 2^logs that starts at global stage sbase; `part` = segment index).
template <int R>
__device__ __forceinline__ void fwd_pass(uint64_t* sm, int logs, int ls0, int sbase, int part,
                                         const Twiddle* __restrict__ tw, uint64_t q, uint64_t q2,
                                         bool last) {
  constexpr int G = 1 << R;
  const int lt = logs - ls0 - R;  // log2 of the element distance inside a group
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
      constexpr int dummy = 0;
      (void)dummy;
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

// Inverse GS pass over R stages (local stages ls0 .. ls0+R-1; element
// distance 2^ls0).  `final_scale`: the pass holds the last global stage,
// which is merged with the n^-1 scaling and canonicalisation.
template <int R>
__device__ __forceinline__ void inv_pass(uint64_t* sm, int logs, int ls0, int logn, int part,
                                         const Twiddle* __restrict__ tw, const LimbConst& c,
                                         bool final_scale, bool canon) {
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
      const int s = ls0 + u;  // global inverse stage (segments start at stage 0)
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

// Pass plan: last pass takes min(5, logs) stages, the rest split evenly.
__device__ __forceinline__ int pass_count(int logs) {
  int rem = logs - (logs < 5 ? logs : 5);
  return 1 + (rem + 4) / 5;
}
__device__ __forceinline__ int pass_size(int logs, int p, int np) {
  int last = logs < 5 ? logs : 5;
  if (p == np - 1) return last;
  int rem = logs - last, k = np - 1;
  int base = rem / k, extra = rem % k;
  return base + (p < extra ? 1 : 0);
}

template <bool FWD>
__global__ void __launch_bounds__(512) ntt_smem_kernel(uint64_t* __restrict__ data, int64_t n_segs,
                                                       int logs, int logn, int period, int offset,
                                                       const LimbConst* __restrict__ lcs,
                                                       const Twiddle* __restrict__ tws) {
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
    if (S >= 2) {
      const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(p);
      for (int i = threadIdx.x; i < S / 2; i += blockDim.x) {
        ulonglong2 v = p2[i];
        sm[phys(2 * i)] = v.x;
        sm[phys(2 * i + 1)] = v.y;
      }
    }
    __syncthreads();
    const int np = pass_count(logs);
    if (FWD) {
      int ls = 0;
      for (int pi = 0; pi < np; ++pi) {
        const int R = pass_size(logs, pi, np);
        const bool last = pi == np - 1;
        switch (R) {
          case 1: fwd_pass<1>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
          case 2: fwd_pass<2>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
          case 3: fwd_pass<3>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
          case 4: fwd_pass<4>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
          default: fwd_pass<5>(sm, logs, ls, logn - logs, part, tw, c.q, c.q2, last); break;
        }
        ls += R;
        __syncthreads();
      }
    } else {
      // inverse: small distances first -> run the plan mirrored
      int ls = 0;
      const bool final_scale = logs == logn;
      for (int pi = np - 1; pi >= 0; --pi) {
        const int R = pass_size(logs, pi, np);
        const bool canon = pi == 0;
        switch (R) {
          case 1: inv_pass<1>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
          case 2: inv_pass<2>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
          case 3: inv_pass<3>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
          case 4: inv_pass<4>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
          default: inv_pass<5>(sm, logs, ls, logn, part, tw, c, final_scale, canon); break;
        }
        ls += R;
        __syncthreads();
      }
    }
    ulonglong2* o2 = reinterpret_cast<ulonglong2*>(p);
    for (int i = threadIdx.x; i < S / 2; i += blockDim.x) {
      ulonglong2 v;
      v.x = sm[phys(2 * i)];
      v.y = sm[phys(2 * i + 1)];
      o2[i] = v;
    }
    __syncthreads();
  }
}

// Forward stage 0 of an n > 16384 row in global memory: (a_j, a_{j+n/2}) with psi[1].
__global__ void ntt_fwd_stage0(uint64_t* __restrict__ data, int64_t n_rows, int logn, int period,
                               int offset, const LimbConst* __restrict__ lcs,
                               const Twiddle* __restrict__ tws) {
  const int n = 1 << logn, h = n >> 1;
  const int64_t total = n_rows * h;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
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

// Inverse last stage of an n > 16384 row: merged with n^-1, canonical out.
__global__ void ntt_inv_last(uint64_t* __restrict__ data, int64_t n_rows, int logn, int period,
                             int offset, const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn, h = n >> 1;
  const int64_t total = n_rows * h;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / h;
    const int j = (int)(e % h);
    const LimbConst c = lcs[offset + (int)(row % period)];
    uint64_t* p = data + row * n;
    uint64_t X = p[j], Y = p[j + h];
    p[j] = shoup(X + Y, c.ninv, c.ninv_s, c.q);
    p[j + h] = shoup(X - Y + c.q2, c.wlast, c.wlast_s, c.q);
  }
}

static int ntt_threads(int logs) {
  int S = 1 << logs;
  int t = S / 32;
  if (t < 32) t = 32;
  if (t > 512) t = 512;
  return t;
}

static size_t ntt_smem_bytes(int logs) {
  int S = 1 << logs;
  return (size_t)(S + S / 32 + 2) * sizeof(uint64_t);
}

static const int kMaxLogS = 14;

static int set_smem_attr() {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    size_t mx = ntt_smem_bytes(kMaxLogS);
    cudaError_t e1 = cudaFuncSetAttribute(ntt_smem_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    cudaError_t e2 = cudaFuncSetAttribute(ntt_smem_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    err = e1 != cudaSuccess ? e1 : e2;
  });
  if (err != cudaSuccess) return check_cuda(err, "cudaFuncSetAttribute(ntt)");
  return FCN_OK;
}

int launch_ntt(const fcn_ring* r, uint64_t* d, int64_t n_rows, int period, int offset, bool fwd,
               cudaStream_t st) {
  if (n_rows <= 0) return FCN_OK;
  int rc = set_smem_attr();
  if (rc) return rc;
  const int logn = r->logn;
  const int logs = logn < kMaxLogS ? logn : kMaxLogS;
  const int64_t segs = n_rows << (logn - logs);
  const int threads = ntt_threads(logs);
  const size_t smem = ntt_smem_bytes(logs);
  int dev_sms = 148;
  int64_t grid = segs;
  const int64_t cap = (int64_t)dev_sms * 64;
  if (grid > cap) grid = cap;
  if (fwd) {
    if (logs < logn) {
      ntt_fwd_stage0<<<grid_for(n_rows << (logn - 1), 256), 256, 0, st>>>(d, n_rows, logn, period, offset,
                                                                           r->d_lc, r->d_fwd);
      FCN_LAUNCH_CHECK("ntt_fwd_stage0");
    }
    ntt_smem_kernel<true><<<(int)grid, threads, smem, st>>>(d, segs, logs, logn, period, offset, r->d_lc,
                                                            r->d_fwd);
    FCN_LAUNCH_CHECK("ntt_smem_kernel<fwd>");
  } else {
    ntt_smem_kernel<false><<<(int)grid, threads, smem, st>>>(d, segs, logs, logn, period, offset, r->d_lc,
                                                             r->d_inv);
    FCN_LAUNCH_CHECK("ntt_smem_kernel<inv>");
    if (logs < logn) {
      ntt_inv_last<<<grid_for(n_rows << (logn - 1), 256), 256, 0, st>>>(d, n_rows, logn, period, offset,
                                                                         r->d_lc);
      FCN_LAUNCH_CHECK("ntt_inv_last");
    }
  }
  return FCN_OK;
}

// ------------------------------------------------------- elementwise ops

template <int OP>
__global__ void binary_kernel(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                              uint64_t* __restrict__ out, int64_t total, int logn, int period, int offset,
                              int64_t b_words, const LimbConst* __restrict__ lcs) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int limb = offset + (int)((e >> logn) % period);
    const uint64_t q = lcs[limb].q;
    const uint64_t x = a[e];
    uint64_t r;
    if (OP == FCN_OP_NEG) {
      r = x ? q - x : 0;
    } else {
      const uint64_t y = b[e % b_words];
      if (OP == FCN_OP_ADD) r = addmod(x, y, q);
      else if (OP == FCN_OP_SUB) r = submod(x, y, q);
      else r = mulmod(x, y, lcs[limb]);
    }
    out[e] = r;
  }
}

// Signed integers -> residues: out[b][l][j] = vals[b][j] mod q_(offset+l).
__global__ void lift_signed_kernel(const int64_t* __restrict__ vals, uint64_t* __restrict__ out, int64_t total,
                                   int logn, int limbs, int offset, const LimbConst* __restrict__ lcs) {
  const int n = 1 << logn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e >> logn;
    const int j = (int)(e & (n - 1));
    const int64_t b = row / limbs;
    const int l = (int)(row % limbs);
    const LimbConst c = lcs[offset + l];
    const int64_t v = vals[(b << logn) + j];
    const uint64_t mag = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
    const uint64_t r = shoup(mag, 1, c.one_s, c.q);
    out[e] = (v < 0 && r) ? c.q - r : r;
  }
}

struct ScalarArgs {
  uint64_t w[64];
  uint64_t ws[64];
};

__global__ void scalar_kernel(const uint64_t* __restrict__ a, uint64_t* __restrict__ out, int64_t total,
                              int logn, int period, int offset, const LimbConst* __restrict__ lcs,
                              ScalarArgs sa) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int li = (int)((e >> logn) % period);
    out[e] = shoup(a[e], sa.w[li], sa.ws[li], lcs[offset + li].q);
  }
}

__global__ void monomial_kernel(const uint64_t* __restrict__ a, uint64_t* __restrict__ out, int64_t total,
                                int logn, int k, int period, int offset, const LimbConst* __restrict__ lcs,
                                ScalarArgs sa) {
  const int n = 1 << logn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e >> logn;
    const int j = (int)(e & (n - 1));
    const int li = (int)(row % period);
    const uint64_t q = lcs[offset + li].q;
    int src = j - k;
    bool wrap = src < 0;
    if (wrap) src += n;
    uint64_t v = shoup(a[(row << logn) + src], sa.w[li], sa.ws[li], q);
    out[e] = (wrap && v) ? q - v : v;
  }
}

}  // namespace fcn

using namespace fcn;

// ----------------------------------------------------------------- C ABI

extern "C" const char* fcn_last_error(void) { return g_last_error.c_str(); }
extern "C" int fcn_version(void) { return 1; }
extern "C" long long fcn_launch_count(void) { return g_launches.load(); }

extern "C" int fcn_ring_create(int device, int n, int count, const uint64_t* primes, fcn_ring** out) {
  if (!out || !primes || count <= 0 || count > 64) return set_error(FCN_ERR_ARG, "bad ring arguments");
  if (n < 4 || n > 32768 || (n & (n - 1))) return set_error(FCN_ERR_PARAM, "ring degree %d is not a power of two in [4, 32768]", n);
  fcn_ring* r = new fcn_ring();
  r->device = device;
  r->n = n;
  r->logn = bitlen64((uint64_t)n) - 1;
  r->L = count;
  std::vector<Twiddle> fw((size_t)count * n), iv((size_t)count * n);
  for (int l = 0; l < count; ++l) {
    const uint64_t q = primes[l];
    if (q >= (1ull << 62) || !h_is_prime(q)) {
      delete r;
      return set_error(FCN_ERR_PARAM, "limb modulus %llu is not a prime below 2^62", (unsigned long long)q);
    }
    uint64_t root;
    if (!root_2n(q, n, &root)) {
      delete r;
      return set_error(FCN_ERR_PARAM, "limb modulus %llu is not = 1 (mod %d)", (unsigned long long)q, 2 * n);
    }
    const uint64_t iroot = h_powmod(root, q - 2, q);
    r->primes.push_back(q);
    r->roots.push_back(root);
    std::vector<uint64_t> pw(n), ipw(n);
    pw[0] = ipw[0] = 1;
    for (int i = 1; i < n; ++i) {
      pw[i] = h_mulmod(pw[i - 1], root, q);
      ipw[i] = h_mulmod(ipw[i - 1], iroot, q);
    }
    for (int i = 0; i < n; ++i) {
      const uint32_t j = bitrev((uint32_t)i, r->logn);
      Twiddle a{pw[j], h_shoup(pw[j], q)};
      Twiddle b{ipw[j], h_shoup(ipw[j], q)};
      fw[(size_t)l * n + i] = a;
      iv[(size_t)l * n + i] = b;
    }
    r->host_lc.push_back(make_limb_const(q, n, iv[(size_t)l * n + 1].w));
  }
  DeviceGuard g(device);
  cudaError_t e = cudaMalloc(&r->d_lc, sizeof(LimbConst) * count);
  if (e == cudaSuccess) e = cudaMalloc(&r->d_fwd, sizeof(Twiddle) * fw.size());
  if (e == cudaSuccess) e = cudaMalloc(&r->d_inv, sizeof(Twiddle) * iv.size());
  if (e == cudaSuccess) e = cudaMemcpy(r->d_lc, r->host_lc.data(), sizeof(LimbConst) * count, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(r->d_fwd, fw.data(), sizeof(Twiddle) * fw.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(r->d_inv, iv.data(), sizeof(Twiddle) * iv.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    fcn_ring_destroy(r);
    return check_cuda(e, "fcn_ring_create upload");
  }
  *out = r;
  return FCN_OK;
}

extern "C" int fcn_ring_destroy(fcn_ring* r) {
  if (!r) return FCN_OK;
  {
    DeviceGuard g(r->device);
    cudaFree(r->d_lc);
    cudaFree(r->d_fwd);
    cudaFree(r->d_inv);
  }
  delete r;
  return FCN_OK;
}

extern "C" int fcn_ring_roots(const fcn_ring* r, uint64_t* roots_out) {
  if (!r || !roots_out) return set_error(FCN_ERR_ARG, "null argument");
  for (int i = 0; i < r->L; ++i) roots_out[i] = r->roots[i];
  return FCN_OK;
}

static int check_rows(const fcn_ring* r, int64_t n_rows, int period, int offset) {
  if (!r) return set_error(FCN_ERR_ARG, "null ring");
  if (n_rows < 0 || period <= 0 || offset < 0 || offset + period > r->L)
    return set_error(FCN_ERR_ARG, "row/limb selection out of range (period %d offset %d limbs %d)", period, offset, r->L);
  return FCN_OK;
}

extern "C" int fcn_ntt_forward(const fcn_ring* r, uint64_t* d, int64_t n_rows, int period, int offset,
                               void* stream) {
  int rc = check_rows(r, n_rows, period, offset);
  if (rc) return rc;
  DeviceGuard g(r->device);
  return launch_ntt(r, d, n_rows, period, offset, true, (cudaStream_t)stream);
}

extern "C" int fcn_ntt_inverse(const fcn_ring* r, uint64_t* d, int64_t n_rows, int period, int offset,
                               void* stream) {
  int rc = check_rows(r, n_rows, period, offset);
  if (rc) return rc;
  DeviceGuard g(r->device);
  return launch_ntt(r, d, n_rows, period, offset, false, (cudaStream_t)stream);
}

extern "C" int fcn_poly_binary(const fcn_ring* r, int op, const uint64_t* a, const uint64_t* b, int64_t b_rows,
                               uint64_t* out, int64_t n_rows, int period, int offset, void* stream) {
  int rc = check_rows(r, n_rows, period, offset);
  if (rc) return rc;
  if (op < 0 || op > 3) return set_error(FCN_ERR_ARG, "unknown op %d", op);
  if (!a || !out || (op != FCN_OP_NEG && !b)) return set_error(FCN_ERR_ARG, "null operand");
  if (op != FCN_OP_NEG && (b_rows <= 0 || b_rows > n_rows || n_rows % b_rows || b_rows % period))
    return set_error(FCN_ERR_ARG, "b_rows %lld must divide n_rows %lld and be a multiple of the limb period", (long long)b_rows, (long long)n_rows);
  const int64_t total = n_rows << r->logn;
  if (!total) return FCN_OK;
  const int64_t bw = (op == FCN_OP_NEG ? n_rows : b_rows) << r->logn;
  DeviceGuard g(r->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = grid_for(total, 256);
  switch (op) {
    case FCN_OP_ADD: binary_kernel<FCN_OP_ADD><<<grid, 256, 0, st>>>(a, b, out, total, r->logn, period, offset, bw, r->d_lc); break;
    case FCN_OP_SUB: binary_kernel<FCN_OP_SUB><<<grid, 256, 0, st>>>(a, b, out, total, r->logn, period, offset, bw, r->d_lc); break;
    case FCN_OP_NEG: binary_kernel<FCN_OP_NEG><<<grid, 256, 0, st>>>(a, b, out, total, r->logn, period, offset, bw, r->d_lc); break;
    default: binary_kernel<FCN_OP_MUL><<<grid, 256, 0, st>>>(a, b, out, total, r->logn, period, offset, bw, r->d_lc); break;
  }
  FCN_LAUNCH_CHECK("binary_kernel");
  return FCN_OK;
}

static int make_scalar_args(const fcn_ring* r, const uint64_t* c_res, int period, int offset, ScalarArgs* sa) {
  if (!c_res) return set_error(FCN_ERR_ARG, "null scalar residues");
  if (period > 64) return set_error(FCN_ERR_ARG, "too many limbs for scalar op");
  for (int i = 0; i < period; ++i) {
    const uint64_t q = r->primes[offset + i];
    const uint64_t w = c_res[i] % q;
    sa->w[i] = w;
    sa->ws[i] = h_shoup(w, q);
  }
  return FCN_OK;
}

extern "C" int fcn_scalar_mul(const fcn_ring* r, const uint64_t* a, const uint64_t* c_res, uint64_t* out,
                              int64_t n_rows, int period, int offset, void* stream) {
  int rc = check_rows(r, n_rows, period, offset);
  if (rc) return rc;
  ScalarArgs sa;
  rc = make_scalar_args(r, c_res, period, offset, &sa);
  if (rc) return rc;
  const int64_t total = n_rows << r->logn;
  if (!total) return FCN_OK;
  DeviceGuard g(r->device);
  scalar_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(a, out, total, r->logn, period, offset,
                                                                        r->d_lc, sa);
  FCN_LAUNCH_CHECK("scalar_kernel");
  return FCN_OK;
}

extern "C" int fcn_poly_mul_monomial(const fcn_ring* r, const uint64_t* a, int k, const uint64_t* c_res,
                                     uint64_t* out, int64_t n_rows, int period, int offset, void* stream) {
  int rc = check_rows(r, n_rows, period, offset);
  if (rc) return rc;
  if (k < 0 || k >= r->n) return set_error(FCN_ERR_ARG, "monomial exponent %d out of [0, %d)", k, r->n);
  if (a == out) return set_error(FCN_ERR_ARG, "monomial multiply cannot run in place");
  ScalarArgs sa;
  rc = make_scalar_args(r, c_res, period, offset, &sa);
  if (rc) return rc;
  const int64_t total = n_rows << r->logn;
  if (!total) return FCN_OK;
  DeviceGuard g(r->device);
  monomial_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(a, out, total, r->logn, k, period,
                                                                          offset, r->d_lc, sa);
  FCN_LAUNCH_CHECK("monomial_kernel");
  return FCN_OK;
}

extern "C" int fcn_lift_signed(const fcn_ring* r, const int64_t* d_vals, int64_t count, uint64_t* d_out, int limbs,
                               int offset, void* stream) {
  int rc = check_rows(r, count, limbs, offset);
  if (rc) return rc;
  if (!d_vals || !d_out) return set_error(FCN_ERR_ARG, "null buffer");
  const int64_t total = (count * limbs) << r->logn;
  if (!total) return FCN_OK;
  DeviceGuard g(r->device);
  lift_signed_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(d_vals, d_out, total, r->logn, limbs, offset,
                                                                             r->d_lc);
  FCN_LAUNCH_CHECK("lift_signed_kernel");
  return FCN_OK;
}
