// k_gemm_tc.cu — tcgen05 tensor-core GEMM (placeholder until the TMA/TMEM kernel lands).
#include "kernels.h"

namespace rh {

bool GemmTcSupported(const GemmArgs&) { return false; }

void LaunchGemmTc(const GemmArgs&, cudaStream_t) { Fail("tcgen05 GEMM not built", RH_ERR_UNSUPPORTED); }

}  // namespace rh
