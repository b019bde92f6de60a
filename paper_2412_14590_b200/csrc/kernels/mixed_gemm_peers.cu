// mixed_gemm_peers.cu — the fused-gather K2 instantiations (PEER = 1,
// mq_mixed_linear_peers): every output element also goes to the peer ranks'
// outputs. Its own translation unit: built in parallel with the plain kernels.
#include "mixed_gemm_sm100.cuh"

namespace mq {

cudaError_t launch_mixed_gemm_tc_peers(const GemmParams& p, int token_tile, int mode, bool pdl, cudaStream_t stream) {
    return launch_tc<1>(p, token_tile, mode, pdl, stream);
}

}  // namespace mq
