// gemm_tc.h — tcgen05/TMEM bf16 grouped expert GEMMs (gemm_tc.cu).
#pragma once

#include <cuda.h>

#include "kernels.h"

namespace moe {

bool tc_row_gemm_supported(const RowGemmArgs& a);
void launch_row_gemm_tc(const RowGemmArgs& a, cudaStream_t st);
bool tc_wgrad_gemm_supported(const WgradGemmArgs& a);
void launch_wgrad_gemm_tc(const WgradGemmArgs& a, cudaStream_t st);
// Force the SIMT path for bf16 as well (testing / A-B comparisons).
void tc_set_enabled(bool on);
bool tc_enabled();

namespace tc {
// 2D TMA tensor map over [rows, cols] row-major elements of `esz` bytes
CUtensorMap make_map_2d(const void* base, CUtensorMapDataType dt, int esz, int64_t rows, int64_t cols,
                        int box_cols, int box_rows, bool swizzle128);
CUtensorMap make_map_2d_swz(const void* base, CUtensorMapDataType dt, int esz, int64_t rows, int64_t cols,
                            int box_cols, int box_rows, int swizzle_bytes);
}  // namespace tc

}  // namespace moe
