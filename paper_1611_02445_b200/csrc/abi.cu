// C ABI housekeeping: version, thread-local error, device selection and the
// host-visible copy of the compiled-in lattice/layout tables.
#include <cstring>

#include "common.cuh"
#include "d3q19.cuh"

namespace tlbm {

static thread_local char g_error[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_error, sizeof(g_error), fmt, ap);
    va_end(ap);
}

}  // namespace tlbm

using namespace tlbm;

extern "C" int tlbm_abi_version(void) { return TLBM_ABI_VERSION; }

extern "C" const char *tlbm_last_error(void) { return g_error; }

extern "C" int tlbm_set_device(int device) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur == device) return TLBM_OK;
    return cuda_check(cudaSetDevice(device), "cudaSetDevice");
}

extern "C" int tlbm_lattice_tables(int table, int32_t *h_e, int32_t *h_opp,
                                   double *h_w, int32_t *h_perm) {
    int rc = check_table(table);
    if (rc) return rc;
    for (int q = 0; q < Q; ++q) {
        if (h_e) {
            h_e[3 * q + 0] = ex(q);
            h_e[3 * q + 1] = ey(q);
            h_e[3 * q + 2] = ez(q);
        }
        if (h_opp) h_opp[q] = opp(q);
        if (h_w) h_w[q] = weight(q);
        if (h_perm)
            for (int j = 0; j < 64; ++j)
                h_perm[64 * q + j] = layout_slot(kind_of(table, q), j & 3, (j >> 2) & 3, j >> 4);
    }
    return TLBM_OK;
}

extern "C" int tlbm_set_l2_fetch_granularity(int bytes) {
    return cuda_check(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes),
                      "cudaDeviceSetLimit(MaxL2FetchGranularity)");
}

extern "C" int tlbm_get_l2_fetch_granularity(int *bytes) {
    size_t v = 0;
    int rc = cuda_check(cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity),
                        "cudaDeviceGetLimit(MaxL2FetchGranularity)");
    if (!rc) *bytes = (int)v;
    return rc;
}
