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
#include <map>
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

cudaError_t kernel_occupancy(const void* fn, int threads, size_t smem, int* occ_out) {
  struct Key {
    const void* fn;
    int dev, threads;
    size_t smem;
    bool operator<(const Key& o) const {
      if (fn != o.fn) return fn < o.fn;
      if (dev != o.dev) return dev < o.dev;
      if (threads != o.threads) return threads < o.threads;
      return smem < o.smem;
    }
  };
  static std::mutex mu;
  static std::map<Key, int> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const Key key{fn, dev, threads, smem};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *occ_out = it->second;
      return cudaSuccess;
    }
  }
  if (smem > 48 * 1024) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) occ = 1;
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = occ;
  *occ_out = occ;
  return cudaSuccess;
}

int device_sms() {
  static std::mutex mu;
  static std::map<int, int> sms;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lk(mu);
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) v = 148;
  sms[dev] = v;
  return v;
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
  c.nq = (uint64_t)0 - q;
  const unsigned __int128 m = (((unsigned __int128)1) << 64) / q;
  c.m32 = (m >> 32) ? 0u : (uint32_t)m;
  c.fq = (double)q;
  c.fqi = 1.0 / (double)q;
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
  std::vector<Twiddle> fw((size_t)count * n), iv((size_t)count * n), ict((size_t)count * n), tws((size_t)count * n);
  std::vector<Twiddle> fl((size_t)count * n);
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
    // DIT inverse: stage s (pairs 2^s apart) uses W_s^k = psi^-(k n / 2^s) at [2^s + k];
    // the final twist multiplies output j by n^-1 psi^-j.
    const uint64_t ninv = h_powmod((uint64_t)n % q, q - 2, q);
    ict[(size_t)l * n] = Twiddle{1, h_shoup(1, q)};
    for (int sg = 0; (1 << sg) < n; ++sg)
      for (int k = 0; k < (1 << sg); ++k) {
        const uint64_t w = ipw[(size_t)k * (n >> sg)];
        ict[(size_t)l * n + (1 << sg) + k] = Twiddle{w, h_shoup(w, q)};
      }
    for (int j = 0; j < n; ++j) {
      const uint64_t w = h_mulmod(ninv, ipw[j], q);
      tws[(size_t)l * n + j] = Twiddle{w, h_shoup(w, q)};
    }
    if (n >= 32) {
      const int T = n / 32;
      size_t o = (size_t)l * n;
      for (int u = 0; u < 5; ++u) {
        const int s0 = (r->logn - 5) + u;
        for (int blk = 0; blk < (1 << u); ++blk)
          for (int t = 0; t < T; ++t) fl[o++] = fw[(size_t)l * n + (1 << s0) + ((size_t)t << u) + blk];
      }
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
  if (e == cudaSuccess) e = cudaMalloc(&r->d_ict, sizeof(Twiddle) * ict.size());
  if (e == cudaSuccess) e = cudaMalloc(&r->d_twist, sizeof(Twiddle) * tws.size());
  if (e == cudaSuccess) e = cudaMemcpy(r->d_ict, ict.data(), sizeof(Twiddle) * ict.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(r->d_twist, tws.data(), sizeof(Twiddle) * tws.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&r->d_fwd_last, sizeof(Twiddle) * fl.size());
  if (e == cudaSuccess) e = cudaMemcpy(r->d_fwd_last, fl.data(), sizeof(Twiddle) * fl.size(), cudaMemcpyHostToDevice);
  // FP64 tables for the limbs below 2^51 (entries of larger limbs stay zero)
  r->fp_ok = true;
  for (int l = 0; l < count; ++l) r->fp_ok &= primes[l] < (1ull << 51);
  {
    const std::vector<Twiddle>* src[4] = {&fw, &ict, &tws, &fl};
    double2** dst[4] = {&r->d_ffwd, &r->d_fict, &r->d_ftwist, &r->d_ffl};
    std::vector<double2> f((size_t)count * n);
    for (int tb = 0; tb < 4 && e == cudaSuccess; ++tb) {
      for (int l = 0; l < count; ++l) {
        const uint64_t q = primes[l];
        for (int i = 0; i < n; ++i) {
          const size_t o = (size_t)l * n + i;
          if (q >= (1ull << 51) || (tb == 3 && n < 32)) {
            f[o] = make_double2(0.0, 0.0);
            continue;
          }
          const uint64_t w = (*src[tb])[o].w;
          const double ws = w > q / 2 ? -(double)(q - w) : (double)w;
          f[o] = make_double2(ws, ws / (double)q);
        }
      }
      e = cudaMalloc(dst[tb], sizeof(double2) * f.size());
      if (e == cudaSuccess) e = cudaMemcpy(*dst[tb], f.data(), sizeof(double2) * f.size(), cudaMemcpyHostToDevice);
    }
  }
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
    cudaFree(r->d_ict);
    cudaFree(r->d_twist);
    cudaFree(r->d_fwd_last);
    cudaFree(r->d_ffwd);
    cudaFree(r->d_fict);
    cudaFree(r->d_ftwist);
    cudaFree(r->d_ffl);
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
