// mixed_gemm_sm100.cu — the plain K2 kernels (PEER = 0) and the launch entry;
// the kernel itself is mixed_gemm_sm100.cuh, the fused-gather instantiations
// are compiled separately (mixed_gemm_peers.cu).
#include "mixed_gemm_sm100.cuh"

namespace mq {

cudaError_t launch_mixed_gemm_tc_peers(const GemmParams& p, int token_tile, int mode, bool pdl, cudaStream_t stream);

int gemm_stages(int bn) {
    switch (bn) {
        case 16: return TcCfg<16>::NS;
        case 32: return TcCfg<32>::NS;
        case 64: return TcCfg<64>::NS;
        default: return TcCfg<128>::NS;
    }
}

cudaError_t launch_mixed_gemm_tc(const GemmParams& p, int token_tile, int mode, bool pdl, cudaStream_t stream) {
    if (p.npeer > 1) return launch_mixed_gemm_tc_peers(p, token_tile, mode, pdl, stream);
    return launch_tc<0>(p, token_tile, mode, pdl, stream);
}

}  // namespace mq
