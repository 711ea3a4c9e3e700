// FP64-pipe instruction-mix microbenchmark on B200: are DADD / DMUL / DFMA
// issued at the same rate, and does the NTT butterfly's mix (2 DMUL, 2 DFMA,
// 3 DADD, 1 FRND) run faster when its additions are written as DFMA?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dpmix tools/dpmix.cu && ./build/dpmix
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 12
template <int OP>
__global__ void __launch_bounds__(256) k_op(double* out, double seed, int reps) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = seed * (threadIdx.x + c + 1);
  const double m = 1.0000001, k = 0.3;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) a[c] = fma(a[c], m, k);
      else if (OP == 1) a[c] = a[c] + k;
      else if (OP == 2) a[c] = a[c] * m;
      else if (OP == 3) {  // 1:1:1 mix
        if (c % 3 == 0) a[c] = fma(a[c], m, k);
        else if (c % 3 == 1) a[c] = a[c] + k;
        else a[c] = a[c] * m;
      } else if (OP == 4) a[c] = rint(a[c]) + k;  // FRND + DADD
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// V 0: the kernel's butterfly.  V 1: additions as DFMA.  V 2: quotient by the
// magic constant.  V 3: Y' = fma(-2, t, X').
template <int V>
__device__ __forceinline__ void bfly(double& X, double& Y, double w, double wq, double q, double one) {
  const double a = Y;
  const double h = a * w;
  const double l = fma(a, w, -h);
  double qt;
  if (V == 2) {
    const double M = 6755399441055744.0;
    qt = fma(a, wq, M) - M;
  } else {
    qt = rint(a * wq);
  }
  const double x = X;
  if (V == 1) {
    const double t = fma(l, one, fma(-qt, q, h));
    X = fma(t, one, x);
    Y = fma(-t, one, x);
  } else if (V == 3) {
    const double t = fma(-qt, q, h) + l;
    X = x + t;
    Y = fma(-2.0, t, X);
  } else {
    const double t = fma(-qt, q, h) + l;
    X = x + t;
    Y = x - t;
  }
}

__device__ __forceinline__ double redq(double x, double qi, double q) {
  const double M = 6755399441055744.0;
  const double qt = fma(x, qi, M) - M;
  return fma(-qt, q, x);
}

template <int V, int MINB>
__global__ void __launch_bounds__(256, MINB) k_bfly(double* out, const double2* __restrict__ tw, double q, int reps, double one) {
  double x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (double)((threadIdx.x * 131 + j * 7) % 1000003) - 500000.0;
  const double qi = 1.0 / q;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int s = 0; s < 15; ++s) {
      const int u = s % 5;
      if (s == 7) {
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
          bfly<V>(x[j], x[j + h], w.x, w.y, q, one);
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
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  double* o;
  cudaMalloc(&o, sizeof(double) * sms * 8 * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 4096;
  const char* names[5] = {"DFMA", "DADD", "DMUL", "DFMA:DADD:DMUL", "FRND+DADD"};
  for (int op = 0; op < 5; ++op) {
    auto launch = [&] {
      if (op == 0) k_op<0><<<sms * 4, 256>>>(o, 1.0, reps);
      if (op == 1) k_op<1><<<sms * 4, 256>>>(o, 1.0, reps);
      if (op == 2) k_op<2><<<sms * 4, 256>>>(o, 1.0, reps);
      if (op == 3) k_op<3><<<sms * 4, 256>>>(o, 1.0, reps);
      if (op == 4) k_op<4><<<sms * 4, 256>>>(o, 1.0, reps);
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
    printf("%-16s %.3f T iter/s (%.1f per SM per clk @1.965GHz)\n", names[op], ops / (ms * 1e-3) / 1e12,
           ops / (ms * 1e-3) / sms / 1.965e9);
  }
  const double q = 1125899906842624.0 + 3 * 32768.0 + 1.0;  // ~2^50 (value only; primality is irrelevant here)
  double2 h[64];
  for (int i = 0; i < 64; ++i) {
    double w = (double)((1234567ll * (i + 3) * 7919ll) % (long long)q);
    if (w > q / 2) w -= q;
    h[i] = make_double2(w, w / q);
  }
  double2* d;
  cudaMalloc(&d, sizeof(h));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const char* nm[4] = {"kernel butterfly", "adds as DFMA", "magic quotient", "Y' = fma(-2,t,X')"};
  for (int mb = 1; mb <= 2; ++mb)
    for (int v = 0; v < 4; ++v) {
      const int br = 86;
      auto launch = [&] {
        if (mb == 2) {
          if (v == 0) k_bfly<0, 2><<<sms * 2, 256>>>(o, d, q, br, 1.0);
          if (v == 1) k_bfly<1, 2><<<sms * 2, 256>>>(o, d, q, br, 1.0);
          if (v == 2) k_bfly<2, 2><<<sms * 2, 256>>>(o, d, q, br, 1.0);
          if (v == 3) k_bfly<3, 2><<<sms * 2, 256>>>(o, d, q, br, 1.0);
        } else {
          if (v == 0) k_bfly<0, 1><<<sms, 256>>>(o, d, q, br, 1.0);
          if (v == 1) k_bfly<1, 1><<<sms, 256>>>(o, d, q, br, 1.0);
          if (v == 2) k_bfly<2, 1><<<sms, 256>>>(o, d, q, br, 1.0);
          if (v == 3) k_bfly<3, 1><<<sms, 256>>>(o, d, q, br, 1.0);
        }
      };
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int i = 0; i < 5; ++i) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bf = 5.0 * sms * mb * 256.0 * br * 16 * 15;
      printf("butterfly, %d CTA/SM (%s): %.3f T/s (%.2f per SM per clk)  err=%s\n", mb, nm[v], bf / (ms * 1e-3) / 1e12,
             bf / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
