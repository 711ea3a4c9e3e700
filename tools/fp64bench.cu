// FP64-pipe microbenchmarks on B200: raw DFMA / FRND / F2I / I2F throughput
// and a signed-residue FP64 modular multiply (error-free product + rounded
// quotient), to size an FP64 variant of the NTT butterfly against the
// integer mulw (profiles/int_peak.json).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
template <int OP>
__global__ void __launch_bounds__(256) k_op(double* out, double seed, int reps) {
  double a[CH];
  long long ia[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { a[c] = seed * (threadIdx.x + c + 1); ia[c] = threadIdx.x * 3 + c; }
  const double m = 1.0000001, k = 0.3;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) a[c] = fma(a[c], m, k);                 // DFMA
      else if (OP == 1) a[c] = rint(a[c] * m);             // DMUL + FRND
      else if (OP == 2) { ia[c] = __double2ll_rn(a[c]); a[c] = a[c] * m + (double)(ia[c] & 1); }  // F2I + DFMA + I2F
      else if (OP == 3) { ia[c] = ia[c] * 0x9E3779B97F4A7C15ll + 1; }  // 64-bit IMAD (lo)
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c] + (double)ia[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// signed FP64 modmul: r == a*w (mod q), |r| <= 1.5 q for |a| < 2^53, |w| <= q/2
__device__ __forceinline__ double mulq(double a, double w, double wq, double q) {
  const double h = a * w;
  const double l = fma(a, w, -h);
  const double qt = rint(a * wq);
  return fma(-qt, q, h) + l;
}
__device__ __forceinline__ double mulq_magic(double a, double w, double wq, double q) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  const double h = a * w;
  const double l = fma(a, w, -h);
  const double qt = fma(a, wq, M) - M;  // |a*wq| < 2^51
  return fma(-qt, q, h) + l;
}
__device__ __forceinline__ double redq(double x, double qi, double q) {
  const double M = 6755399441055744.0;
  const double qt = fma(x, qi, M) - M;
  return fma(-qt, q, x);
}

// 15 stages per iteration (three 5-stage register passes), values reduced
// before every third stage (RS 0) or once, before stage 7 (RS 1) -- the NTT
// kernels' schedules (ntt_f64.cuh; RS 1 is what limbs just above 2^50 get)
template <int MAGIC, int RS>
__global__ void __launch_bounds__(256, 2) k_bfly(double* out, const double2* __restrict__ tw, double q, int reps) {
  double x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (double)((threadIdx.x * 131 + j * 7) % 1000003) - 500000.0;
  const double qi = 1.0 / q;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int s = 0; s < 15; ++s) {
      const int u = s % 5;
      if (RS == 0 ? (s > 0 && s % 3 == 0) : s == 7) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = redq(x[j], qi, q);
      }
      const int h = 32 >> (u + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << u); ++blk) {
        const double2 w = __ldg(tw + (1 << u) + blk);
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int j = blk * 2 * h + jj;
          const double t = MAGIC ? mulq_magic(x[j + h], w.x, w.y, q) : mulq(x[j + h], w.x, w.y, q);
          const double X = x[j];
          x[j] = X + t;
          x[j + h] = X - t;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = redq(x[j], qi, q);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, sizeof(double) * sms * 4 * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 4096;
  const char* names[4] = {"DFMA", "DMUL+FRND", "F2I+DFMA+I2F", "IMAD64lo"};
  for (int op = 0; op < 4; ++op) {
    auto launch = [&] {
      if (op == 0) k_op<0><<<sms * 4, 256>>>(o, 1.0, reps);
      if (op == 1) k_op<1><<<sms * 4, 256>>>(o, 1.0, reps);
      if (op == 2) k_op<2><<<sms * 4, 256>>>(o, 1.0, reps);
      if (op == 3) k_op<3><<<sms * 4, 256>>>(o, 1.0, reps);
    };
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 3.0 * sms * 4 * 256.0 * reps * CH;
    printf("%-14s %.3f T iter/s (%.1f per SM per clk @1.965GHz)\n", names[op], ops / (ms * 1e-3) / 1e12,
           ops / (ms * 1e-3) / sms / 1.965e9);
  }
  const double q = 2251799813554177.0;  // < 2^51
  double2 h[64];
  for (int i = 0; i < 64; ++i) {
    double w = (double)((1234567ll * (i + 3)) % 2251799813554177ll);
    if (w > q / 2) w -= q;
    h[i] = make_double2(w, w / q);
  }
  double2* d;
  cudaMalloc(&d, sizeof(h));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int v = 0; v < 3; ++v) {  // rint RS0, magic RS0, rint RS1
    const int br = 86;
    auto launch = [&] {
      if (v == 0) k_bfly<0, 0><<<sms * 2, 256>>>(o, d, q, br);
      else if (v == 1) k_bfly<1, 0><<<sms * 2, 256>>>(o, d, q, br);
      else k_bfly<0, 1><<<sms * 2, 256>>>(o, d, q / 2, br);  // RS 1 needs q ~ 2^50
    };
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bf = 5.0 * sms * 2 * 256.0 * br * 16 * 15;
    const char* nm[3] = {"rint, RS0", "magic, RS0", "rint, RS1"};
    printf("fp64 butterfly (%s): %.3f T/s (%.2f per SM per clk)  err=%s\n", nm[v], bf / (ms * 1e-3) / 1e12,
           bf / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
