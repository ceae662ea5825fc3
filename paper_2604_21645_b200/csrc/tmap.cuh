// tmap.cuh -- 2-D TMA tensor maps over row-major fp32 matrices (host side).
// cuTensorMapEncodeTiled is resolved once through the runtime's driver entry
// point (no libcuda link).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.cuh"

namespace pqg {

// rows x ld fp32, box = box_rows x box_cols (box_cols * 4 <= 128 for the
// 128-byte swizzle); rows past `rows` read as zeros
inline bool encode_rows_map(CUtensorMap* m, const float* base, uint64_t rows, uint64_t ld, uint32_t box_rows,
                            uint32_t box_cols, CUtensorMapSwizzle sw) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cuuint64_t(ld), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace pqg
