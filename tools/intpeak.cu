// Integer-pipe microbenchmark (B200): throughput of IMAD, IMAD.WIDE and of
// the NTT's approximate-quotient Shoup product `mulw`, with many independent
// chains per thread so latency is hidden.  Prints ops/s per kind.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1811_09953_b200/csrc/fcn_common.cuh"

using namespace fcn;
#ifndef CH_N
#define CH_N 8
#endif
constexpr int CH = CH_N;   // independent chains per thread
constexpr int ITERS = 4096;

__global__ void k_imad(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= x[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_wide(uint64_t* out, uint32_t a) {
  uint64_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = (uint64_t)(uint32_t)x[c] * a + x[c];  // IMAD.WIDE.U32 with 64-bit addend
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= x[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_imadhi(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __umulhi(x[c], a) + x[c];
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= x[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_mulw(uint64_t* out, uint64_t w, uint64_t ws, uint64_t nq) {
  uint64_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 77 + c;
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = mulw(x[c], w, ws, nq);
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= x[c];
  if (s == 0x12345) out[0] = s;
}

#include <cstdlib>
int main(int argc, char** argv) {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void* buf;
  cudaMalloc(&buf, 64);
  const int bps = argc > 1 ? atoi(argv[1]) : 8;
  const int blocks = sms * bps, threads = 256;
  printf("blocks/SM %d, chains/thread %d\n", bps, CH);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double threads_total = (double)blocks * threads;
  auto run = [&](const char* name, double ops_per_thread, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = ops_per_thread * threads_total * 10;
    printf("%-10s %.3f Tops/s  (%.1f per SM per clk @1.965GHz)\n", name, ops / (ms * 1e-3) / 1e12,
           ops / (ms * 1e-3) / sms / 1.965e9);
  };
  run("imad", (double)ITERS * CH, [&] { k_imad<<<blocks, threads>>>((uint32_t*)buf, 3, 5); });
  run("imad.hi", (double)ITERS * CH, [&] { k_imadhi<<<blocks, threads>>>((uint32_t*)buf, 0x9E3779B9u, 5); });
  run("imad.wide", (double)ITERS * CH, [&] { k_wide<<<blocks, threads>>>((uint64_t*)buf, 3); });
  const uint64_t q = 36028797018972161ull;
  const uint64_t w = 1234567891234567ull % q;
  const uint64_t ws = (uint64_t)(((unsigned __int128)w << 64) / q);
  run("mulw", (double)(ITERS / 8) * CH, [&] { k_mulw<<<blocks, threads>>>((uint64_t*)buf, w, ws, (uint64_t)0 - q); });
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
