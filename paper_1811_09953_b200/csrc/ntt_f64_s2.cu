// libfcn: FP64 NTT kernels, reduction schedule RS = 2 (see ntt_f64.cuh).
#include "ntt_f64.cuh"

namespace fcn {
template int launch_ntt_f64<2>(const fcn_ring*, uint64_t*, int64_t, int, int, bool, cudaStream_t, const uint64_t*, int,
                                 const NttEpi*, int);
template int launch_ntt_f64_sq<2>(const fcn_ring*, const uint64_t*, const uint64_t*, uint64_t*, int64_t, int, int,
                                    cudaStream_t, int, bool);
template int launch_ntt_f64_pair<2>(const fcn_ring*, uint64_t*, int64_t, bool, cudaStream_t, const PairEpi*, int);
}  // namespace fcn
