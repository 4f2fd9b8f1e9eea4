// gemm_tc.h — tcgen05/TMEM bf16 grouped expert GEMMs (gemm_tc.cu).
#pragma once

#include "kernels.h"

namespace moe {

bool tc_row_gemm_supported(const RowGemmArgs& a);
void launch_row_gemm_tc(const RowGemmArgs& a, cudaStream_t st);
bool tc_wgrad_gemm_supported(const WgradGemmArgs& a);
void launch_wgrad_gemm_tc(const WgradGemmArgs& a, cudaStream_t st);
// Force the SIMT path for bf16 as well (testing / A-B comparisons).
void tc_set_enabled(bool on);
bool tc_enabled();

}  // namespace moe
