// tcgen05.mma kind::i8 issue-rate microbenchmark (one CTA per SM, garbage
// operands in shared memory, accumulators in TMEM): clocks per MMA for
// M = 128, K = 32 and N in {64, 128, 256}, A from shared memory (SS) or
// TMEM (TS), no-swizzle canonical layouts as in csrc/mac_tc.cu.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mmabench tools/mmabench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  if (threadIdx.x == 0) {
    const uint32_t A = smem_u32(smem), B = A + 16384;
    const uint64_t ad = sdesc(A, 128, 1024);
    const uint64_t bd = sdesc(B, N * 8, 128);
    if (TS) asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 448), "l"(ad));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)((i & 3) * (N <= 64 ? 64 : 0));
      if (TS)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                     "r"(tmem + 448), "l"(bd), "r"(idesc), "r"(1));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// the kernel's pattern: per 64-input chunk 7 planes x 2 K-steps, A/B at
// distinct shared-memory addresses, accumulators p * 64; SW = 0 no swizzle,
// 64 = SWIZZLE_64B (layout type 4) with the 64-byte atoms
// MODE bit 0: per-chunk tcgen05.commit to a stage barrier (like the kernel);
// bit 1: the other warps spin on an mbarrier until the MMA lane is done
template <int SW, int MODE = 0, int NN = 64, int PL = 7>
__global__ void __launch_bounds__(448, 1) bench_rot(int chunks, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __shared__ __align__(8) uint64_t stage_bar[5];
  __shared__ __align__(8) uint64_t done_bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    for (int i = 0; i < 5; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&stage_bar[i])));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 16) | ((uint32_t)(64 >> 3) << 17) | (8u << 24);
  if (MODE & 4) {  // random operand bytes instead of whatever the shared memory held
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    uint32_t x = 0x9E3779B9u * (threadIdx.x + 1);
    for (int i = threadIdx.x; i < 5 * 36864 / 4; i += blockDim.x) {
      x ^= x << 13;
      x ^= x >> 17;
      x ^= x << 5;
      w[i] = x;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  __shared__ __align__(8) uint64_t full_bar[5], empty_bar[5];
  if (MODE & 8) {
    if (threadIdx.x == 0)
      for (int i = 0; i < 5; ++i) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full_bar[i])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty_bar[i])));
      }
    __syncthreads();
    if (threadIdx.x == 32) {  // producer: refill a stage once the MMAs released it
      for (int c = 0; c < chunks; ++c) {
        const int st = c % 5;
        if (c >= 5) {
          uint32_t ok = 0;
          const uint32_t par = ((c / 5) + 1) & 1;
          while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&empty_bar[st])), "r"(par));
        }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full_bar[st])) : "memory");
      }
    }
  }
  if ((MODE & 2) && threadIdx.x >= 32) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&done_bar)));
  }
  if (threadIdx.x == 0) {
    const uint32_t base = smem_u32(smem);
    long long t0 = clock64();
    for (int c = 0; c < chunks; ++c) {
      if (MODE & 8) {
        uint32_t ok = 0;
        const uint32_t par = (c / 5) & 1;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&full_bar[c % 5])), "r"(par));
      }
      if (MODE & 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&stage_bar[c % 5])));
      const uint32_t A = base + (c % 4) * 45056, B = A + 8192;
      for (int p = 0; p < PL; ++p)
        for (int ks = 0; ks < 2; ++ks) {
          uint64_t ad, bd;
          if (SW == 0) {
            ad = sdesc(A + ks * 256, 128, 512);
            bd = sdesc(B + p * (NN * 64) + ks * (NN * 32), NN * 8, 128);
          } else {
            ad = sdesc(A + ks * 32, 16, 512) | (4ull << 61);
            bd = sdesc(B + p * 4096 + ks * 2048, 4096, 512) | (4ull << 61);
          }
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + p * NN),
                       "l"(ad), "l"(bd), "r"(idesc), "r"(1));
        }
      if (MODE & 8)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&empty_bar[c % 5])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done_bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int SW, int MODE = 0, int NN = 64, int PL = 7>
void run_rot(long long* d, int threads = 128, int chunks = 2048) {
  const int smem = 5 * 36864 + 1024;
  cudaFuncSetAttribute(bench_rot<SW, MODE, NN, PL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench_rot<SW, MODE, NN, PL><<<148, threads, smem>>>(8, d);
  cudaError_t err = cudaDeviceSynchronize();
  bench_rot<SW, MODE, NN, PL><<<148, threads, smem>>>(chunks, d);
  err = cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("rotating operands, %s, %d threads, mode %d, N=%d x %d planes, %d chunks: %.2f clk/MMA, %.1f clk per 64x128 K-chunk-plane (%s)\n",
         SW ? "SWIZZLE_64B" : "no swizzle", threads, MODE, NN, PL, chunks, (double)cyc / (chunks * PL * 2),
         (double)cyc / (chunks * PL * 2) * 64.0 / NN, cudaGetErrorString(err));
}

template <int N, bool TS>
void run(long long* d) {
  const int smem = 16384 + 256 * 128 + 1024;
  cudaFuncSetAttribute(bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  bench<N, TS><<<148, 128, smem>>>(16, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<N, TS><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double macs = 128.0 * N * 32 * iters * 148;
  printf("N=%3d %s: %.2f clk/MMA  %.1f TMAC/s (%s)\n", N, TS ? "TS" : "SS", (double)cyc / iters, macs / (ms * 1e-3) / 1e12,
         cudaGetErrorString(err));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, false>(d);
  run<64, true>(d);
  run<128, false>(d);
  run<128, true>(d);
  run<256, false>(d);
  run<256, true>(d);
  run_rot<0>(d);
  run_rot<64>(d);
  run_rot<0, 0>(d, 448);
  run_rot<0, 1>(d, 128);
  run_rot<0, 2>(d, 448);
  run_rot<0, 3>(d, 448);
  run_rot<0, 4>(d, 128);
  run_rot<0, 7>(d, 448);
  run_rot<0, 12>(d, 128);
  run_rot<0, 14>(d, 448);
  run_rot<0, 12, 128, 4>(d, 128);
  run_rot<0, 12, 256, 2>(d, 128);
  run_rot<0, 4, 128, 4>(d, 128);
  run_rot<0, 4, 256, 2>(d, 128);
  return 0;
}
