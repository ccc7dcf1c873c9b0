// Shared host-side helpers of the C ABI: thread-local error string, launch
// checking and dtype/model/table dispatch.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include "tlbm.h"

namespace tlbm {

void set_error(const char *fmt, ...);

inline int cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return TLBM_ERR_CUDA;
    }
    return TLBM_OK;
}

inline int launch_check(const char *what) {
    return cuda_check(cudaGetLastError(), what);
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int check_dtype(int dtype) {
    if (dtype != TLBM_F64 && dtype != TLBM_F32) {
        set_error("unknown dtype %d", dtype);
        return TLBM_ERR_ARG;
    }
    return TLBM_OK;
}
inline int check_fluid(int fluid) {
    if (fluid != TLBM_INCOMPRESSIBLE && fluid != TLBM_QUASI) {
        set_error("unknown fluid model %d", fluid);
        return TLBM_ERR_ARG;
    }
    return TLBM_OK;
}
inline int check_table(int table) {
    if (table < TLBM_TABLE_XYZ || table > TLBM_TABLE_B200) {
        set_error("unknown layout table %d", table);
        return TLBM_ERR_ARG;
    }
    return TLBM_OK;
}

// Calls f.template operator()<T, QUASI, TABLE>() for the runtime triple.
template <class F>
int dispatch(int dtype, int fluid, int table, F &&f) {
    int rc;
    if ((rc = check_dtype(dtype)) || (rc = check_fluid(fluid)) || (rc = check_table(table)))
        return rc;
#define TLBM_D3(T, QU, TB) \
    if (dtype == (sizeof(T) == 8 ? TLBM_F64 : TLBM_F32) && fluid == QU && table == TB) \
        return f.template operator()<T, QU, TB>();
#define TLBM_D2(T, QU) TLBM_D3(T, QU, 0) TLBM_D3(T, QU, 1) TLBM_D3(T, QU, 2)
    TLBM_D2(double, 0) TLBM_D2(double, 1) TLBM_D2(float, 0) TLBM_D2(float, 1)
#undef TLBM_D2
#undef TLBM_D3
    return TLBM_ERR_ARG;
}

inline unsigned grid_for(long long n, int block) {
    return static_cast<unsigned>((n + block - 1) / block);
}

}  // namespace tlbm
