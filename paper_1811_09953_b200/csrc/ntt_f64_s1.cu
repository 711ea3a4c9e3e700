// libfcn: FP64 NTT kernels, reduction schedule RS = 1 (see ntt_f64.cuh).
#include "ntt_f64.cuh"

namespace fcn {
template int launch_ntt_f64<1>(const fcn_ring*, uint64_t*, int64_t, int, int, bool, cudaStream_t, const uint64_t*, int,
                                 const NttEpi*, int);
template int launch_ntt_f64_sq<1>(const fcn_ring*, const uint64_t*, const uint64_t*, uint64_t*, int64_t, int, int,
                                    cudaStream_t, int, bool);
template int launch_ntt_f64_pair<1>(const fcn_ring*, uint64_t*, int64_t, bool, cudaStream_t, const PairEpi*, int);
}  // namespace fcn

#ifdef FCN_NTT_PROF
// the symbol is per translation unit: the bench shapes run schedule RS = 1 (this unit)
extern "C" int fcn_ntt_prof_read(unsigned long long* out16, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out16, fcn::fcn_ntt_prof, sizeof(unsigned long long) * 16);
  if (e == cudaSuccess && reset) {
    unsigned long long z[16] = {};
    e = cudaMemcpyToSymbol(fcn::fcn_ntt_prof, z, sizeof(z));
  }
  return e == cudaSuccess ? 0 : -1;
}
#endif
