// tcgen05 flash attention (forward + backward) for sm_100a.  (in progress)
#include "attn.h"
#include "gemm.cuh"

namespace mgv {
bool attn_tc_supported(int hd, int Nk) {
    (void)hd;
    (void)Nk;
    return false;
}
void attn_fwd_tc(const AttnProblem&, cudaStream_t) { throw std::runtime_error("attn_fwd_tc not built"); }
void attn_bwd_tc(const AttnBwdProblem&, cudaStream_t) { throw std::runtime_error("attn_bwd_tc not built"); }
}  // namespace mgv
