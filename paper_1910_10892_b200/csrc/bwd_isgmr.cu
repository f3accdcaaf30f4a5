// ISGMR instantiations of the warp-specialised backward (bwd_split.cuh).
#include "bwd_launch.cuh"

namespace mrf {
cudaError_t launch_bwd_isgmr(const AccArgs& a, int batch, cudaStream_t s) { return launch_bwd_sweep<false>(a, batch, s); }
}  // namespace mrf
