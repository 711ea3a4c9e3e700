// Does an integer-pipe NTT butterfly stream overlap an FP64-pipe one on the
// same SM?  Half the CTAs run the FP64 butterfly loop (fp64bench.cu), half
// the integer one (bflybench.cu); compare the mixed rate with each alone.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1811_09953_b200/csrc/fcn_common.cuh"
using namespace fcn;

__device__ __forceinline__ void ibfly(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t ws, uint64_t nq, uint64_t q4) {
  const uint64_t t = mulw(Y, w, ws, nq);
  const uint64_t x = X;
  X = x + t;
  Y = x + q4 - t;
}

__device__ void int_body(uint64_t* out, const ulonglong2* __restrict__ tw, uint64_t q, int reps) {
  uint64_t x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (threadIdx.x * 131 + j * 7) % q;
  const uint64_t nq = 0 - q, q4 = 4 * q;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const int h = 32 >> (u + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << u); ++blk) {
        const ulonglong2 v = __ldg(tw + (1 << u) + blk);
#pragma unroll
        for (int jj = 0; jj < h; ++jj) ibfly(x[blk * 2 * h + jj], x[blk * 2 * h + jj + h], v.x, v.y, nq, q4);
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = csub(x[j], 16 * q);
  }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) s ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ void fp_body(uint64_t* out, const double2* __restrict__ tw, double q, int reps) {
  double x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (double)((threadIdx.x * 131 + j * 7) % 1000003) - 500000.0;
  const double qi = 1.0 / q;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      if (s == 3) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = fredq(x[j], qi, q);
      }
      const int h = 32 >> (s + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << s); ++blk) {
        const double2 w = __ldg(tw + (1 << s) + blk);
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int j = blk * 2 * h + jj;
          const double t = fmulq(x[j + h], w.x, w.y, q);
          const double X = x[j];
          x[j] = X + t;
          x[j + h] = X - t;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fredq(x[j], qi, q);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint64_t)__double_as_longlong(s);
}

// mode 0: all fp, 1: all int, 2: first half of the grid fp, second half int
__global__ void __launch_bounds__(256, 2) k_mix(uint64_t* out, const double2* ftw, const ulonglong2* itw, double fq,
                                                uint64_t iq, int reps_f, int reps_i, int mode) {
  const bool fp = mode == 0 || (mode == 2 && blockIdx.x < gridDim.x / 2);
  if (fp) fp_body(out, ftw, fq, reps_f);
  else int_body(out, itw, iq, reps_i);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double fq = 2251799813554177.0;
  const uint64_t iq = 2251799813554177ull;
  double2 hf[64];
  ulonglong2 hi[64];
  for (int i = 0; i < 64; ++i) {
    uint64_t w = (1234567ull * (i + 3)) % iq;
    double ws = (double)w;
    if (ws > fq / 2) ws -= fq;
    hf[i] = make_double2(ws, ws / fq);
    hi[i] = make_ulonglong2(w, (uint64_t)(((unsigned __int128)w << 64) / iq));
  }
  double2* df;
  ulonglong2* di;
  cudaMalloc(&df, sizeof(hf));
  cudaMalloc(&di, sizeof(hi));
  cudaMemcpy(df, hf, sizeof(hf), cudaMemcpyHostToDevice);
  cudaMemcpy(di, hi, sizeof(hi), cudaMemcpyHostToDevice);
  uint64_t* o;
  cudaMalloc(&o, sizeof(uint64_t) * sms * 2 * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // per-CTA work: reps passes of 80 butterflies per thread
  const int rf = 256, ri = 150;
  const char* names[5] = {"fp64 only", "int only", "mixed 1:1", "fp64 1/SM", "int 1/SM"};
  for (int mode = 0; mode < 5; ++mode) {
    const int g = mode >= 3 ? sms : sms * 2;
    const int mm = mode >= 3 ? mode - 3 : mode;
    k_mix<<<g, 256>>>(o, df, di, fq, iq, rf, ri, mm);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) k_mix<<<g, 256>>>(o, df, di, fq, iq, rf, ri, mm);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bf;
    if (mode == 0) bf = 5.0 * sms * 2 * 256.0 * rf * 80;
    else if (mode == 1) bf = 5.0 * sms * 2 * 256.0 * ri * 80;
    else if (mode == 2) bf = 5.0 * sms * 256.0 * (rf + ri) * 80;
    else if (mode == 3) bf = 5.0 * sms * 256.0 * rf * 80;
    else bf = 5.0 * sms * 256.0 * ri * 80;
    printf("%-10s %.3f ms  %.3f T bfly/s (%.2f /SM/clk)  err=%s\n", names[mode], ms / 5, bf / (ms * 1e-3) / 1e12,
           bf / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
