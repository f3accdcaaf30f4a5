// TRWP instantiations of the warp-specialised backward (bwd_split.cuh).
#include "bwd_launch.cuh"

namespace mrf {
cudaError_t launch_bwd_trwp(const AccArgs& a, int batch, cudaStream_t s) { return launch_bwd_sweep<true>(a, batch, s); }
}  // namespace mrf
