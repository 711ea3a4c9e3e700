// libfcn: the fused sparse power-of-two linear layer on the 5th-generation
// tensor cores (tcgen05 kind::i8, accumulators in TMEM).
//
// Replaces, for SIMD-batched plans, the chain the reference evaluates per
// output (engine.py:698-717: fv.mul_pt with a constant plaintext + fv.add_ct,
// fv.py:439-460 / 394-403):  out[o] = sum_t c_ot * in[i_t]  (mod q_l, every
// coefficient of both polys of every limb).
//
// Exactness: a residue x < 2^(8P) is the sum of its P bytes x_b 2^(8b).  With
// signed 8-bit weights c (|c| <= 127) the tensor cores compute, per byte plane
// b, the exact int32 sums S_b = sum_t c_t x_{t,b} (|S_b| < K 127 255 < 2^31),
// and the epilogue folds V = sum_b S_b 2^(8b) (an exact 128-bit value) into
// V mod q_l.  Nothing is rounded, so the result equals the reference's chain
// of modular products and additions residue for residue.
//
// Data flow:
//   split_planes_kernel : the layer's input ciphertexts [I][2][k][n] u64 ->
//                         byte planes [I][P][2kn] u8 (one pass, coalesced);
//   mac_tc_kernel       : persistent CTAs (one per SM) over the tiles
//                         (output group g, 64-column tile j).
//     warps 0-3  producers: per K-chunk of 64 inputs, cp.async gathers each
//                input's 64-byte plane segments into the MN-major canonical
//                B layout, thread 0 issues one cp.async.bulk (TMA) of the
//                group's pre-laid-out weight tile (K-major canonical A);
//                5-6 stage mbarrier ring (full / empty) of 64-input chunks;
//     warp 4     TMEM owner and MMA issuer: one lane issues P x 4
//                tcgen05.mma.cta_group::1.kind::i8 (M=128, N=64, K=32) per
//                chunk into P TMEM accumulators (64 columns each),
//                tcgen05.commit's each stage back to the producers and the
//                finished tile to the epilogue (tmem_full);
//     warps 5-12 epilogue: tcgen05.ld of their 32 TMEM lanes (= output rows; two
//                warps per lane quarter, 32 columns each),
//                byte-plane fold, reduction mod q_l, u64 stores (+ fan-out),
//                then tmem_empty -- overlapping the next tile's loads.
// Output groups: up to 128 output rows (any set: a dense layer's consecutive
// outputs, or every channel at a few spatial positions of a convolution)
// with the union of their inputs as the K list (built by the host,
// engine._lower_tc).

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "fcn_common.cuh"

namespace fcn {

namespace tc {

constexpr int kChunk = 64;   // inputs (K bytes) per stage
constexpr int kN = 64;       // output columns per CTA tile
constexpr int kM = 128;      // output rows per group
constexpr int kABytes = kM * kChunk;        // 8 KB: K-major weight tile
constexpr int kBPlaneBytes = kN * kChunk;   // 4 KB per byte plane: MN-major
constexpr int kLoadsPerThread = kChunk / 32;  // inputs per producer thread per chunk
constexpr int kRing = 16;  // chunks of input indices staged ahead by the index warp
constexpr int kProducers = 128;             // warps 0-3

// canonical no-swizzle ("interleave") layouts of tcgen05 shared-memory operands
//   A, K-major:  byte (m, k) at (m/8)*1024 + (k/16)*128 + (m%8)*16 + k%16
//                (core matrix 8 rows x 16 B; LBO = 128 B along K, SBO = 1024 B along M)
//   B, MN-major: byte (n, k) at (n/16)*128 + (k/8)*512 + (k%8)*16 + n%16
//                (core matrix 16 columns x 8 K-rows; SBO = 128 B along N, LBO = 512 B along K)
constexpr uint32_t kALbo = 128, kASbo = (kChunk / 16) * 128;
constexpr uint32_t kBSbo = 128, kBLbo = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // start address, LBO, SBO in 16-byte units; version 1 (Blackwell); no swizzle
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// instruction descriptor: D s32, A s8 (K-major), B u8 (MN-major), M = 128, N = 64
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (0u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(kN >> 3) << 17) |
                            ((uint32_t)(kM >> 4) << 24);

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
// for the warps off the MMA critical path: back off between polls, so that
// spinning warps do not steal the shared-memory bandwidth the tensor cores
// read their operands with (measured: 126 -> ~60 clk per MMA issue)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  unsigned ns = 32;
  while (!mbar_try(bar, parity)) {
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : 256;
  }
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// arrive on an mbarrier once all of this thread's prior cp.async have completed
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
// A from TMEM (K-major: row m in lane m, 32 K-bytes per 8 columns), B from shared memory
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
// shared memory (matrix descriptor) -> TMEM: 128 rows x 256 bits into lanes 0..127
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 8 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "r"(taddr));
}
__device__ __forceinline__ void st_global_v4(uint64_t* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace tc

// Byte planes of a batch of rows: planes[r][b][c] = byte b of in[r][c].
// A thread takes 8 consecutive columns of one row (4 x 16-byte loads) and
// writes 8 bytes per plane.
template <int P>
__global__ void __launch_bounds__(256) split_planes_kernel(const uint64_t* __restrict__ in, int64_t rows, int64_t cols,
                                                           uint8_t* __restrict__ planes) {
  const int64_t pitch = tc_plane_pitch(cols);
  const int64_t groups = cols >> 3;
  const int64_t total = rows * groups;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / groups, g8 = e - r * groups;
    const uint4* src = reinterpret_cast<const uint4*>(in + r * cols + (g8 << 3));
    uint4 a = __ldg(src), b = __ldg(src + 1), c = __ldg(src + 2), d = __ldg(src + 3);
    // words: value v = (lo, hi): a = (v0.lo, v0.hi, v1.lo, v1.hi), ...
    const uint32_t lo[8] = {a.x, a.z, b.x, b.z, c.x, c.z, d.x, d.z};
    const uint32_t hi[8] = {a.y, a.w, b.y, b.w, c.y, c.w, d.y, d.w};
    uint8_t* dst = planes + (r * P) * pitch + (g8 << 3);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint32_t* w = p < 4 ? lo : hi;
      const uint32_t s = (uint32_t)(p & 3);
      // byte s of w[0..3] -> one word, byte s of w[4..7] -> another
      const uint32_t sel = s | ((s + 4) << 4);
      const uint32_t x01 = __byte_perm(w[0], w[1], sel), x23 = __byte_perm(w[2], w[3], sel);
      const uint32_t x45 = __byte_perm(w[4], w[5], sel), x67 = __byte_perm(w[6], w[7], sel);
      const uint32_t lo4 = __byte_perm(x01, x23, 0x5410), hi4 = __byte_perm(x45, x67, 0x5410);
      *reinterpret_cast<uint2*>(dst + p * pitch) = make_uint2(lo4, hi4);
    }
  }
}

// Persistent CTAs (one per SM) walk the tiles t = (group g = t % G, column
// tile j = t / G): tiles resident at the same time share their column tile,
// so a column slab's byte planes are read from HBM once and from L2 by the
// other groups.  Warps 0-3 load, warp 4 owns TMEM and issues the MMAs, warps
// 5-12 drain the accumulators (two warps per lane quarter); the epilogue of tile i
// overlaps the loads of tile i+1 and its MMAs wait only for the accumulator
// to be drained (tmem_empty).
__device__ unsigned long long g_tc_dbg[8];  // FCN_TC_DBG & 64: MMA-thread cycle counters (block 0)

template <int P>
struct TcShape {
  static constexpr int kStageBytes = tc::kABytes + P * tc::kBPlaneBytes;
  static constexpr int kStages = (214 * 1024) / kStageBytes;
  static constexpr int kSmem =
      kStages * kStageBytes + tc::kRing * tc::kChunk * 4 + 8 * (2 * kStages + 2 * tc::kRing + 2) + 16;
  static constexpr int kThreads = 14 * 32;  // 4 producer, 1 MMA, 8 epilogue warps, 1 index warp
  // weights staged in TMEM (tcgen05.cp, two buffers after the P accumulators)
  // instead of read from shared memory by every plane's MMA: measured slower
  // (the copy -> MMA dependency serialises each chunk: 87 vs 55 ms on cfg5's
  // skeleton, FCN_TC_DBG ablation), so off; kept for the A/B
  static constexpr bool kATmem = false;
};

template <int P>
__global__ void __launch_bounds__(TcShape<P>::kThreads, 1)
    mac_tc_kernel(const uint8_t* __restrict__ planes, int64_t cols, int64_t n_groups, int64_t n_tiles,
                  const TcGroup* __restrict__ groups, const int32_t* __restrict__ kidx,
                  const int32_t* __restrict__ rows_tab, const int8_t* __restrict__ wimg, Fanout F, int64_t row_lo,
                  int64_t row_hi, int logn, int k, const LimbConst* __restrict__ lcs, int dbg) {
  using namespace tc;
  using S_ = TcShape<P>;
  constexpr int kSt = S_::kStages;
  extern __shared__ __align__(1024) uint8_t smem[];
  int32_t* kring = reinterpret_cast<int32_t*>(smem + kSt * S_::kStageBytes);  // [kRing][kChunk] input indices
  uint64_t* full = reinterpret_cast<uint64_t*>(kring + kRing * kChunk);
  uint64_t* empty = full + kSt;
  uint64_t* kfull = empty + kSt;
  uint64_t* kempty = kfull + kRing;
  uint64_t* tmem_full = kempty + kRing;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pitch = tc_plane_pitch(cols);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], kProducers + 1);
      mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&kfull[r], 32);
      mbar_init(&kempty[r], kProducers);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 256);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {  // TMEM: P accumulators of 64 columns (P <= 8 -> 512 columns)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------ producers
    // this thread: column block nb = lane % 4 (16 columns), inputs
    // kk_i = (kChunk/4) warp + lane/4 + 8 i: every warp instruction copies eight
    // inputs' contiguous 64-byte segments of one plane.  The input indices
    // come from the index warp's shared-memory ring (filled up to kRing
    // chunks ahead), so no global-load latency sits on this loop.
    const int nb = lane & 3;
    int it = 0;  // chunk counter across tiles (stage / phase)
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const TcGroup G = groups[t % n_groups];
      const int64_t col0 = (t / n_groups) * kN;
      const int nchunks = (G.n_k + kChunk - 1) / kChunk;
      for (int c = 0; c < nchunks; ++c, ++it) {
        const int s = it % kSt;
        const int r = it % kRing;
        if (it >= kSt) mbar_wait_sleep(&empty[s], ((it / kSt) + 1) & 1);
        uint8_t* A = smem + s * S_::kStageBytes;
        uint8_t* B = A + kABytes;
        if (threadIdx.x == 0) {
          if (dbg & 4) {
            mbar_arrive(&full[s]);
          } else {
            mbar_arrive_tx(&full[s], kABytes);
            bulk_g2s(A, wimg + ((int64_t)G.w_off + c) * kABytes, kABytes, &full[s]);
          }
        }
        mbar_wait_sleep(&kfull[r], (it / kRing) & 1);
        int32_t cur[kLoadsPerThread];
#pragma unroll
        for (int i = 0; i < kLoadsPerThread; ++i) {
          const int kk = warp * (kChunk / 4) + (lane >> 2) + 8 * i;
          cur[i] = c * kChunk + kk < G.n_k ? kring[r * kChunk + kk] : -1;
        }
        mbar_arrive(&kempty[r]);
#pragma unroll
        for (int i = 0; i < kLoadsPerThread; ++i) {
          if (cur[i] >= 0 && !(dbg & 1)) {
            const int kk = warp * (kChunk / 4) + (lane >> 2) + 8 * i;
            const uint8_t* src = planes + ((int64_t)cur[i] * P) * pitch + col0 + nb * 16;
            uint8_t* dst = B + (kk >> 3) * kBLbo + (kk & 7) * 16 + nb * kBSbo;
#pragma unroll
            for (int p = 0; p < P; ++p) cp_async16(dst + p * kBPlaneBytes, src + p * pitch);
          }
        }
        // the stage's full barrier completes when this thread's copies have
        // landed (hardware arrive, no producer wait): the producers run
        // ahead by as many chunks as there are stages
        cp_async_arrive_noinc(&full[s]);
      }
    }
  } else if (warp == 13) {
    // ------------------------------------------------------ index warp
    // copies each chunk's 64 input indices (256 bytes, 16-byte aligned: the
    // host pads every group's list to a multiple of 4) into the ring
    int it = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const TcGroup G = groups[t % n_groups];
      const int nchunks = (G.n_k + kChunk - 1) / kChunk;
      for (int c = 0; c < nchunks; ++c, ++it) {
        const int r = it % kRing;
        if (it >= kRing) mbar_wait_sleep(&kempty[r], ((it / kRing) + 1) & 1);
        if (lane < kChunk / 4) cp_async16(kring + r * kChunk + lane * 4, kidx + G.k_off + c * kChunk + lane * 4);
        cp_async_arrive_noinc(&kfull[r]);
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int it = 0, local = 0;
      unsigned long long w_full = 0, w_tmem = 0, t_start = clock64();
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++local) {
        const TcGroup G = groups[t % n_groups];
        const int nchunks = (G.n_k + kChunk - 1) / kChunk;
        unsigned long long c0 = clock64();
        if (local > 0) mbar_wait(tmem_empty, (local - 1) & 1);  // accumulator drained
        w_tmem += clock64() - c0;
        tc_fence_after();
        for (int c = 0; c < nchunks; ++c, ++it) {
          const int s = it % kSt;
          c0 = clock64();
          mbar_wait(&full[s], (it / kSt) & 1);
          w_full += clock64() - c0;
          // the B tiles were written by the producers' cp.async (generic
          // proxy): make them visible to the tensor cores' async-proxy reads
          if (!(dbg & 16)) fence_proxy_async();
          tc_fence_after();
          const uint32_t A = smem_u32(smem + s * S_::kStageBytes);
          const uint32_t B = A + kABytes;
          const int rem = G.n_k - c * kChunk;
          const int ksteps = rem >= kChunk ? kChunk / 32 : (rem + 31) / 32;
          if (S_::kATmem && !(dbg & 8)) {
            // the weight tile goes to TMEM once (tcgen05.cp, 32 bytes per
            // lane per K-step) and the P plane MMAs read it from there: shared
            // memory then only feeds B (2 KB per MMA instead of 6 KB)
            const uint32_t abuf = tmem + P * kN + (uint32_t)(it & 1) * (kChunk / 4);
            for (int ks = 0; ks < ksteps; ++ks) tmem_cp_128x256b(abuf + ks * 8, smem_desc(A + ks * 2 * kALbo, kALbo, kASbo));
#pragma unroll
            for (int p = 0; p < P; ++p) {
              for (int ks = 0; ks < ksteps; ++ks) {
                const uint64_t bd = smem_desc(B + p * kBPlaneBytes + ks * 4 * kBLbo, kBLbo, kBSbo);
                mma_i8_ts(tmem + p * kN, abuf + ks * 8, bd, (c > 0 || ks > 0) ? 1u : 0u);
              }
            }
          } else {
#pragma unroll
            for (int p = 0; p < P; ++p) {
              for (int ks = 0; ks < ksteps; ++ks) {
                const uint64_t ad = smem_desc(A + ks * 2 * kALbo, kALbo, kASbo);
                const uint64_t bd = smem_desc(B + p * kBPlaneBytes + ks * 4 * kBLbo, kBLbo, kBSbo);
                mma_i8(tmem + p * kN, ad, bd, (c > 0 || ks > 0) ? 1u : 0u);
              }
            }
          }
          if (!(dbg & 32) || c == nchunks - 1) mma_commit(&empty[s]);
          else mbar_arrive(&empty[s]);
        }
        mma_commit(tmem_full);
      }
      if ((dbg & 64) && blockIdx.x == 0) {
        g_tc_dbg[0] = clock64() - t_start;
        g_tc_dbg[1] = w_full;
        g_tc_dbg[2] = w_tmem;
        g_tc_dbg[3] = it;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------ epilogue (warps 5-12)
    const int q4 = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 5) >> 2;  // which 32 of the 64 columns
    const int m = q4 * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16);
    int local = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++local) {
      const TcGroup G = groups[t % n_groups];
      const int64_t col0 = (t / n_groups) * kN;
      const int limb = (int)((col0 >> logn) % k);
      const uint64_t q = lcs[limb].q;
      const double qinv = 1.0 / (double)q;
      const bool live = m < G.m;
      const int64_t orow = live ? (int64_t)rows_tab[G.row_off + m] : -1;
      const bool store = live && orow >= row_lo && orow < row_hi;
      const int64_t obase = (orow - row_lo) * cols + col0;
      mbar_wait_sleep(tmem_full, local & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cg = half * (kN / 2); cg < (half + 1) * (kN / 2); cg += 8) {
        int32_t Sv[P][8];
#pragma unroll
        for (int p = 0; p < P; ++p) tmem_ld8(taddr + p * kN + cg, Sv[p]);
        tmem_wait_ld();
        if (cg == (half + 1) * (kN / 2) - 8) {  // all of this thread's words read: release TMEM
          tc_fence_before();
          mbar_arrive(tmem_empty);
        }
        if (dbg & 2) continue;
        uint64_t res[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // V = L + H 2^32, L = sum_{b<4} S_b 2^(8b), H = sum_{b>=4} S_b 2^(8(b-4)); |V| < 2^83
          int64_t L = 0, H = 0;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            if (p < 4)
              L += (int64_t)Sv[p][u] << (8 * p);
            else
              H += (int64_t)Sv[p][u] << (8 * (p - 4));
          }
          // quotient estimate within 1 of V / q (|V| 2^-52 / q < 1/2 for q > 2^32),
          // remainder exact in wrapping 64-bit arithmetic, then two corrections
          const double vd = fma((double)H, 4294967296.0, (double)L);
          const int64_t qh = __double2ll_rn(vd * qinv);
          int64_t r = (int64_t)((uint64_t)L + ((uint64_t)H << 32) - (uint64_t)qh * q);
          r += r < 0 ? (int64_t)q : 0;
          r += r < 0 ? (int64_t)q : 0;
          r -= r >= (int64_t)q ? (int64_t)q : 0;
          r -= r >= (int64_t)q ? (int64_t)q : 0;
          res[u] = (uint64_t)r;
        }
        if (store) {
#pragma unroll
          for (int d = 0; d < kMaxFanout; ++d) {
            if (d < F.n) {
              uint64_t* o = F.dst[d] + obase + cg;  // two 32-byte stores: whole sectors
              st_global_v4(o, res[0], res[1], res[2], res[3]);
              st_global_v4(o + 4, res[4], res[5], res[6], res[7]);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// FCN_TC_DBG (timing ablations only; results are wrong): 1 = producers skip
// the byte-plane gathers, 2 = the epilogue skips the fold and the stores,
// 4 = no weight-tile copies, 8 = weights read from shared memory (SS MMA),
// 16 = no proxy fence before the MMAs, 32 = stages released without tcgen05.commit,
// 64 = print the MMA thread's cycle split (block 0) after the launch
static int tc_debug() {
  static const int v = [] {
    const char* e = getenv("FCN_TC_DBG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int P>
static int launch_tc_t(const TcLaunch& a, cudaStream_t st) {
  using S_ = TcShape<P>;
  int occ = 0;
  FCN_CUDA(kernel_occupancy((const void*)mac_tc_kernel<P>, S_::kThreads, (size_t)S_::kSmem, &occ));
  const int64_t n_tiles = a.n_groups * (a.cols / tc::kN);
  int64_t grid = (int64_t)device_sms();
  if (grid > n_tiles) grid = n_tiles;
  mac_tc_kernel<P><<<(unsigned)grid, S_::kThreads, S_::kSmem, st>>>(a.planes, a.cols, a.n_groups, n_tiles, a.groups,
                                                                    a.kidx, a.rows, a.wimg, a.out, a.row_lo,
                                                                    a.row_hi, a.logn, a.k, a.lcs, tc_debug());
  FCN_LAUNCH_CHECK("mac_tc_kernel");
  if (tc_debug() & 64) {
    unsigned long long h[8];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_tc_dbg, sizeof(h));
    fprintf(stderr, "[mac_tc] block0: %llu clk total, %llu waiting full, %llu waiting tmem_empty, %llu chunks\n", h[0],
            h[1], h[2], h[3]);
  }
  return FCN_OK;
}

int launch_mac_tc(const TcLaunch& a, cudaStream_t st) {
  if (a.n_groups <= 0) return FCN_OK;
  if (a.cols % tc::kN) return set_error(FCN_ERR_ARG, "columns per ciphertext must be a multiple of %d", tc::kN);
  switch (a.planes_n) {
    case 5: return launch_tc_t<5>(a, st);
    case 6: return launch_tc_t<6>(a, st);
    case 7: return launch_tc_t<7>(a, st);
    case 8: return launch_tc_t<8>(a, st);
    default: return set_error(FCN_ERR_PARAM, "tensor-core MAC supports 5..8 byte planes (got %d)", a.planes_n);
  }
}

int launch_split_planes(const uint64_t* in, int64_t rows, int64_t cols, int P, uint8_t* planes, cudaStream_t st) {
  if (rows <= 0) return FCN_OK;
  if (cols % 8) return set_error(FCN_ERR_ARG, "columns must be a multiple of 8");
  const int64_t total = rows * (cols / 8);
  int64_t grid = (total + 255) / 256;
  const int64_t cap = (int64_t)device_sms() * 16;
  if (grid > cap) grid = cap;
  switch (P) {
#define FCN_SP(PP) \
  case PP: split_planes_kernel<PP><<<(unsigned)grid, 256, 0, st>>>(in, rows, cols, planes); break;
    FCN_SP(5) FCN_SP(6) FCN_SP(7) FCN_SP(8)
#undef FCN_SP
    default: return set_error(FCN_ERR_PARAM, "5..8 byte planes (got %d)", P);
  }
  FCN_LAUNCH_CHECK("split_planes_kernel");
  return FCN_OK;
}

}  // namespace fcn
