// gemm_tc.cu -- tcgen05 typed grouped GEMM (placeholder until the tensor-core
// kernel lands; the SIMT kernel in gemm_simt.cu serves every shape meanwhile).
#include "kernels.cuh"

namespace rgnn {
rgnn_status launch_gemm_fwd_tc(int, int, const GemmFwdArgs&, cudaStream_t) { return RGNN_E_UNSUPPORTED; }
}  // namespace rgnn
