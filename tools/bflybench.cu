// Butterfly-throughput microbenchmark: 32 register-resident residues per
// thread, repeated 5-stage Cooley-Tukey passes with the NTT's butterfly
// (mulw + lazy adds), no memory traffic except L1-resident twiddles.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1811_09953_b200/csrc/fcn_common.cuh"
using namespace fcn;

__device__ __forceinline__ void bfly(uint64_t& X, uint64_t& Y, const Twiddle& w, uint64_t nq, uint64_t q4) {
  const uint64_t t = mulw(Y, w.w, w.s, nq);
  const uint64_t x = X;
  X = x + t;
  Y = x + q4 - t;
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_bfly(uint64_t* out, const Twiddle* __restrict__ tw, uint64_t q, int reps) {
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
        const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(tw + (1 << u) + blk));
        const Twiddle w{v.x, v.y};
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int j = blk * 2 * h + jj;
          bfly(x[j], x[j + h], w, nq, q4);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = csub(x[j], 16 * q);  // keep bounded (ALU only)
  }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) s ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main(int argc, char** argv) {
  const int bps = argc > 1 ? atoi(argv[1]) : 2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t q = 36028797018972161ull;
  Twiddle h[64];
  for (int i = 0; i < 64; ++i) {
    uint64_t w = (1234567ull * (i + 3)) % q;
    h[i] = Twiddle{w, (uint64_t)(((unsigned __int128)w << 64) / q)};
  }
  Twiddle* d;
  cudaMalloc(&d, sizeof(h));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  uint64_t* o;
  cudaMalloc(&o, sizeof(uint64_t) * sms * 2 * 256);
  const int reps = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&] {
    if (bps == 1) k_bfly<1><<<sms, 256>>>(o, d, q, reps);
    else k_bfly<2><<<sms * 2, 256>>>(o, d, q, reps);
  };
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bf = 5.0 * sms * bps * 256.0 * reps * 80;
  printf("blocks/SM %d: %.3f T butterflies/s (%.2f per SM per clk @1.965GHz)  err=%s\n", bps, bf / (ms * 1e-3) / 1e12,
         bf / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
