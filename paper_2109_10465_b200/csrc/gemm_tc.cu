// gemm_tc.cu — tcgen05/TMEM bf16 grouped expert GEMMs (placeholder; see below).
#include "common.cuh"
#include "gemm_tc.h"

namespace moe {

static bool g_tc_enabled = true;
void tc_set_enabled(bool on) { g_tc_enabled = on; }
bool tc_row_gemm_supported(const RowGemmArgs&) { return false; }
void launch_row_gemm_tc(const RowGemmArgs&, cudaStream_t) { throw Status(8, "tcgen05 row GEMM not built"); }
bool tc_wgrad_gemm_supported(const WgradGemmArgs&) { return false; }
void launch_wgrad_gemm_tc(const WgradGemmArgs&, cudaStream_t) { throw Status(8, "tcgen05 wgrad GEMM not built"); }

}  // namespace moe
