// The fused D3Q19 step: pull gather through the neighbour-tile map, halfway
// bounce-back fill, BB_WALL reflection, Zou-He inlet/outlet, LBGK collision
// and the store into the other copy -- Alg. 2 of the paper
// with the boundary contract of boundaries.py:1-28.
//
// Work mapping: one tile = 64 threads (2 warps, thread j <-> slot j, i.e. the
// paper's x + 4y + 16z map, lattice.py:97-106); TILES_PER_CTA tiles per CTA.
// Each thread issues its 19 loads back to back (one address select per
// direction: neighbour slot if the link exists, else the node's own opposite
// slot), so 19 independent 8-byte loads per thread are in flight.  Loads use
// the read-only path (the source copy is immutable during the launch) and hit
// L1 when the two warps of a tile share a sector.  With the B200 table every
// 32-byte sector of the source copy is consumed by exactly one destination
// tile, so DRAM traffic is the 2 x 19 x 8 B / node minimum plus metadata
// (4 B/node meta word + 108 B/tile neighbour row).
// (kernel and launch templates: step_impl.cuh; instantiated per dtype in
// step_f64.cu / step_f32.cu; this file validates and dispatches.)
#include "common.cuh"
#include "d3q19.cuh"

namespace tlbm {
int step_launch_f64(const tlbm_step_args *a, cudaStream_t s);
int step_launch_f32(const tlbm_step_args *a, cudaStream_t s);
}  // namespace tlbm

using namespace tlbm;

extern "C" int tlbm_step(const tlbm_step_args *a, void *stream) {
    if (!a) {
        set_error("tlbm_step: null argument");
        return TLBM_ERR_ARG;
    }
    // an empty store (all-solid geometry) has no buffers and nothing to do
    if (a->t_n == 0 && a->tile_begin == 0 && a->tile_end == 0) return TLBM_OK;
    if (!a->f_src || !a->f_dst || !a->meta ||
        (a->variant != TLBM_READ_WRITE_ONLY && !a->nbr)) {
        set_error("tlbm_step: null argument");
        return TLBM_ERR_ARG;
    }
    if (a->f_src == a->f_dst) {
        set_error("tlbm_step: source and destination copies must differ");
        return TLBM_ERR_ARG;
    }
    if (a->tile_begin < 0 || a->tile_end > a->t_n || a->tile_begin > a->tile_end) {
        set_error("tlbm_step: tile range [%lld, %lld) outside [0, %lld)",
                  (long long)a->tile_begin, (long long)a->tile_end, (long long)a->t_n);
        return TLBM_ERR_ARG;
    }
    if (a->collision != TLBM_LBGK && a->collision != TLBM_MRT) {
        set_error("tlbm_step: unknown collision model %d", a->collision);
        return TLBM_ERR_ARG;
    }
    if (a->arith != TLBM_ARITH_REFERENCE && a->arith != TLBM_ARITH_FMA) {
        set_error("tlbm_step: unknown arithmetic mode %d", a->arith);
        return TLBM_ERR_ARG;
    }
    if (a->arith == TLBM_ARITH_FMA && a->dtype != TLBM_F64) {
        // fp32 FMA drifts past the 1e-5 parity bar (u: 1.1e-5 after 1000
        // cavity-64 steps, tests/test_gpu_fma.py), so it is not offered
        set_error("tlbm_step: FMA arithmetic is fp64-only");
        return TLBM_ERR_ARG;
    }
    if (a->collision == TLBM_MRT && !a->mrt_op) {
        set_error("tlbm_step: MRT needs the 19x19 operator (mrt_op)");
        return TLBM_ERR_ARG;
    }
    if (a->collision == TLBM_LBGK && !(a->tau > 0.5)) {
        set_error("tlbm_step: relaxation time must exceed 0.5, got %g", a->tau);
        return TLBM_ERR_ARG;
    }
    if (a->iter_counter && (!a->flags || a->ring_len <= 0)) {
        set_error("tlbm_step: a device iteration counter needs flags and ring_len > 0");
        return TLBM_ERR_ARG;
    }
    int rc;
    if ((rc = check_dtype(a->dtype)) || (rc = check_fluid(a->fluid)) ||
        (rc = check_table(a->table)))
        return rc;
    return a->dtype == TLBM_F64 ? step_launch_f64(a, as_stream(stream))
                                : step_launch_f32(a, as_stream(stream));
}

namespace {
__global__ void advance_counter_kernel(long long *c, long long k) { *c += k; }
}  // namespace

extern "C" int tlbm_advance_counter(int64_t *d_counter, int64_t k, void *stream) {
    if (!d_counter) {
        set_error("tlbm_advance_counter: null counter");
        return TLBM_ERR_ARG;
    }
    advance_counter_kernel<<<1, 1, 0, as_stream(stream)>>>(
        reinterpret_cast<long long *>(d_counter), (long long)k);
    return launch_check("advance_counter_kernel");
}
