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
#pragma once
#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "physics.cuh"

namespace tlbm {
namespace step_detail {

// the MRT operator travels by value in the kernel parameters (constant bank)
// (dense row-major A, or per-column distinct values when grouped: physics.cuh)
template <class T, bool MRT>
struct MrtOperator {
    T op[Q * Q];
    int grouped;   // reference arithmetic: per-column distinct values
};
template <class T>
struct MrtOperator<T, false> {};

template <class T, bool MRT = false>
struct StepParams {
    MrtOperator<T, MRT> mrt;
    const T *__restrict__ src;
    T *__restrict__ dst;
    const int32_t *__restrict__ nbr;
    const uint32_t *__restrict__ meta;
    long long tile_begin, tile_end;
    double inv_tau;
    double inlet_u[3];
    double outlet_rho;
    double guard_sq;        // |u|^2 threshold of the guard (+inf: off)
    uint32_t *flags;
    const long long *iter;  // graph mode: status ring slot read on the device
    long long iter_add;
    unsigned long long ring_len;
    // fused halo: post-collision outgoing z planes also stored into a
    // neighbour's ghost tiles (peer memory), tile t -> dst + (t - begin) * 1216
    T *halo_up;             // e_z = +1 directions of plane z = 3
    long long halo_up_begin, halo_up_end;
    T *halo_down;           // e_z = -1 directions of plane z = 0
    long long halo_down_begin, halo_down_end;
    // compact tile storage (compact.cu, step_compact.cuh); null otherwise
    const long long *__restrict__ cbase;
    const int *__restrict__ cnf;
    const unsigned char *__restrict__ crank;
    // traversal order (may be null = tile order): CTA position -> tile
    const int *__restrict__ order;
    // fused halo on compact storage: neighbour block offsets of its ghosts
    const long long *halo_up_cbase;
    const long long *halo_down_cbase;
    // node-parallel compact step (step_kernel_nodes); node_meta null otherwise
    const uint32_t *__restrict__ node_meta;
    const void *__restrict__ node_rec;
    const int *__restrict__ unit_tile;
    const void *__restrict__ entries;
    long long node_begin, node_end;
    // sizeof(T) and sizeof(uint2) as run-time values: ptxas cannot
    // strength-reduce base + i * scale into a LEA / LEA.HI.X pair (ALU pipe)
    // and keeps one IMAD.WIDE.U32 (FMA pipe) per address (step_kernel_nodes)
    unsigned scale_value, scale_entry;
};

// the tile at launch position pos (tile_begin <= pos < tile_end); ORDERED
// kernels read the traversal order, the others keep the tile-list order
// (a template switch: the extra pointer alone made the fp32 kernel spill)
template <bool ORDERED, class P>
__device__ __forceinline__ long long tile_at(const P &p, long long pos) {
    if constexpr (ORDERED) return (long long)__ldg(p.order + pos);
    else return pos;
}

__host__ __device__ constexpr int up_dir(int k) {
    return k == 0 ? 5 : k == 1 ? 11 : k == 2 ? 13 : k == 3 ? 15 : 17;
}

constexpr int TILE_VALUES = Q * 64;

// Tiles per CTA and the occupancy target (resident warps per SM, which sets
// the register cap through __launch_bounds__), per dtype and collision.
// fp64 LBGK: 2 tiles (128 threads) per CTA at 32 warps/SM (64 registers)
// measured best on B200: 0.797 ms / 256^3 channel step vs 0.915 ms at 4
// tiles / 78 registers and 1.39 ms at 48 warps / 40 registers
// (scripts/step_sweep.py, profiles/).  fp32 LBGK moves half the bytes per
// node, so at 32 warps/SM its loads cannot cover the latency: 64 warps/SM (32
// registers) in 64-thread CTAs takes it from 0.490 to 0.410 ms (0.80 -> 0.95
// of the HBM peak).  MRT keeps 19 deviations live next to the populations.
#ifndef TLBM_TPC
#define TLBM_TPC 2
#endif
#ifndef TLBM_TPC_F32
#define TLBM_TPC_F32 1
#endif
#ifndef TLBM_WARPS
#define TLBM_WARPS 32
#endif
#ifndef TLBM_WARPS_F32
#define TLBM_WARPS_F32 64
#endif
// MRT, reference arithmetic (grouped product, 19 live row sums): at one tile
// per CTA, 20 warps/SM (96 registers, 56 B spill) runs the 256^3 channel in
// 0.979 ms vs 1.029 at 16 (126 registers) and 1.015 at 24; the compact
// kernels gain too (node-parallel 0.721 -> 0.757 at porosity 1.0)
// (scripts/exp/exp62.sh, exp63.sh; at two tiles per CTA 16 had won,
// exp34.sh).  FMA arithmetic: 24 (0.828 ms vs 0.935 at 28).
#ifndef TLBM_WARPS_MRT
#define TLBM_WARPS_MRT 20
#endif
#ifndef TLBM_WARPS_MRT_FMA
#define TLBM_WARPS_MRT_FMA 24
#endif
// fp32 MRT: the block-store kernel (packed row sums, TLBM_MRT_PACKED 2) at
// 32 warps/SM (no spill) 0.586 ms vs 0.623 at 40; with packed products only
// 40 had won (0.624 vs 0.636 at 32); the compact kernels keep 32
// (node-parallel at 40: 0.544 vs 0.593 of peak at porosity 0.2)
// (scripts/exp/exp64.sh, exp71.sh)
#ifndef TLBM_WARPS_MRT_F32
#define TLBM_WARPS_MRT_F32 32
#endif
#ifndef TLBM_WARPS_COMPACT_MRT_F32
#define TLBM_WARPS_COMPACT_MRT_F32 32
#endif

template <class T>
constexpr int tiles_per_cta() { return sizeof(T) == 4 ? TLBM_TPC_F32 : TLBM_TPC; }
// fp64 MRT: one tile per CTA (8 CTAs of 2 warps at 16 warps/SM) staggers the
// CTAs' gather and product phases: 1.032-1.059 vs 1.062-1.071 ms (reference
// arithmetic), 0.827-0.830 vs 0.840 (FMA) on the 256^3 channel; LBGK keeps
// two (scripts/exp/exp60.sh)
#ifndef TLBM_TPC_MRT
#define TLBM_TPC_MRT 1
#endif
template <class T, bool MRT>
constexpr int tiles_per_cta_of() { return MRT && sizeof(T) == 8 ? TLBM_TPC_MRT : tiles_per_cta<T>(); }

// (The 64-bit path's earlier formulation -- 64-bit offsets rebuilt per pull --
// came out of ptxas 12.9 with out-of-bounds addresses at 32 and 40 registers
// (compute-sanitizer, tests/test_gpu_step.py::test_index64_path); the staged
// block pointers below are clean at 32 and run 0.89 of peak in fp32.)
// fp32 propagation-only (bench ladder): 48 warps/SM, 0.416 ms vs 0.441 at 64
#ifndef TLBM_WARPS_PROP_F32
#define TLBM_WARPS_PROP_F32 48
#endif
template <class T, bool MRT, int VARIANT, bool FMA = false>
constexpr int min_blocks() {
    constexpr int warps = sizeof(T) == 4
        ? (MRT ? TLBM_WARPS_MRT_F32
               : (VARIANT == TLBM_PROPAGATION_ONLY ? TLBM_WARPS_PROP_F32 : TLBM_WARPS_F32))
        : (MRT ? (FMA ? TLBM_WARPS_MRT_FMA : TLBM_WARPS_MRT) : TLBM_WARPS);
    return warps / (2 * tiles_per_cta_of<T, MRT>());
}

// TLBM_LOAD_MODE (tuning knob): 0 ld.global.nc (default), 1 ld.global,
// 2 ld.global.nc with an L2 evict_last hint
#ifndef TLBM_LOAD_MODE
#define TLBM_LOAD_MODE 0
#endif
template <class T>
__device__ __forceinline__ T load_ro(const T *p) {
#if TLBM_LOAD_MODE == 1
    T v;
    if constexpr (sizeof(T) == 8)
        asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else
        asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
#elif TLBM_LOAD_MODE == 2
    T v;
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    if constexpr (sizeof(T) == 8)
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
#else
    return __ldg(p);
#endif
}

// Hide how a pointer was formed so the compiler keeps it as one 64-bit
// register (base + 32-bit offset -> a single IMAD.WIDE per access) instead of
// re-deriving src + tile * 1216 + offset for every load.
template <class T>
__device__ __forceinline__ const T *opaque(const T *p) {
    asm("" : "+l"(p));
    return p;
}

template <class T>
__device__ __forceinline__ void store_out(T *p, T v) {
#ifdef TLBM_STORE_CS
    __stcs(p, v);
#else
    *p = v;
#endif
}

// Pull table: for every (direction q, slot j) one packed word --
//   bits  0-10  q*64 + L_q(source slot)        (pulled, in the source tile)
//   bits 11-21  opp(q)*64 + L_opp(q)(j)        (halfway bounce-back, own tile)
//   bits 22-26  neighbour-row index of the source tile delta (13 = own)
// -- built at compile time per layout table (a __device__ constant), so
// each pull costs one L1-resident table load instead of the per-direction
// boundary tests and layout arithmetic.
struct PullTable {
    uint32_t w[Q * 64];
};

template <int TABLE>
constexpr PullTable make_pull_table() {
    PullTable t{};
    for (int q = 0; q < Q; ++q)
        for (int j = 0; j < 64; ++j) {
            const int x = j & 3, y = (j >> 2) & 3, z = j >> 4;
            const int sx = x - ex(q), sy = y - ey(q), sz = z - ez(q);
            const int dx = sx < 0 ? -1 : (sx > 3 ? 1 : 0);
            const int dy = sy < 0 ? -1 : (sy > 3 ? 1 : 0);
            const int dz = sz < 0 ? -1 : (sz > 3 ? 1 : 0);
            const uint32_t pulled = q * 64 + layout_slot(kind_of(TABLE, q), sx & 3, sy & 3, sz & 3);
            const uint32_t bounced = opp(q) * 64 + layout_slot(kind_of(TABLE, opp(q)), x, y, z);
            t.w[q * 64 + j] = pulled | (bounced << 11) | ((uint32_t)delta_index(dx, dy, dz) << 22);
        }
    return t;
}

__device__ const PullTable kPullTables[3] = {make_pull_table<0>(), make_pull_table<1>(),
                                             make_pull_table<2>()};

// REL32: neighbour rows are staged as 32-bit element offsets relative to the
// thread's own tile, so every per-direction address is one 32-bit add/select
// and one IMAD.WIDE from a 64-bit base fixed per thread; valid whenever
// |nbr - tile| * 1216 < 2^31 (checked on the host, tiling.py).  Otherwise
// (e.g. a periodic wrap across more than 1.77 M tiles) the 64-bit path stages
// the 27 neighbour block addresses themselves and selects a pointer per pull.
template <class T, int QUASI, int TABLE, int VARIANT, int TPC, bool REL32, bool MRT, bool HALO,
          bool FMA, bool ORDERED>
__global__ void __launch_bounds__(64 * TPC, min_blocks<T, MRT, VARIANT, FMA>())
step_kernel(const StepParams<T, MRT> p) {
    __shared__ int s_nbr[TPC][NBR];
    __shared__ const T *s_ptr[REL32 ? 1 : TPC][NBR];
    const int ti = threadIdx.x >> 6;
    const int j = threadIdx.x & 63;
    const long long pos0 = p.tile_begin + (long long)blockIdx.x * TPC;
    const bool valid = pos0 + ti < p.tile_end;
    const long long tile = ORDERED ? (valid ? tile_at<ORDERED>(p, pos0 + ti) : 0) : pos0 + ti;

    // Pulls read their packed word through the read-only path (the 4.9 KB
    // table stays L1-resident).  Measured on B200 (scripts/step_sweep.py, at
    // the 32-warp fp32 shape): 0.50 ms vs 0.51-0.56 with per-direction
    // address arithmetic, 0.57 with a per-CTA shared-memory copy (whose 640
    // MB/step of staging loads cost more than they save) and 0.55 with
    // 16-byte unpacked entries (LDG.128: the hoisted 76 registers spill);
    // fp64 unchanged at 0.78 ms.
    //
    // The neighbour row is staged as the tile-index difference to the
    // thread's own tile (0 for the own-tile entry 13); REL32 stores it
    // pre-multiplied by the 1216 values of a tile.
    if (VARIANT != TLBM_READ_WRITE_ONLY) {
        for (int i = threadIdx.x; i < TPC * NBR; i += 64 * TPC) {
            const bool ok = pos0 + i / NBR < p.tile_end;
            const long long t = ORDERED ? (ok ? tile_at<ORDERED>(p, pos0 + i / NBR) : 0)
                                        : pos0 + i / NBR;
            const long long nb = ok ? p.nbr[t * NBR + i % NBR] : -1;
            const long long d = nb >= 0 ? nb - t : 0;
            s_nbr[i / NBR][i % NBR] = (int)(REL32 ? d * TILE_VALUES : d);
            if (!REL32) s_ptr[REL32 ? 0 : i / NBR][i % NBR] = p.src + (t + d) * TILE_VALUES;
        }
        __syncthreads();
    }

    const uint32_t meta = valid ? p.meta[tile * 64 + j] : 0u;
    uint32_t status = 0;
    if (meta & META_ACTIVE) {
        const int x = j & 3, y = (j >> 2) & 3, z = j >> 4;
        const long long own = tile * TILE_VALUES;
        const T *base = opaque(p.src + own);
        T g[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (VARIANT == TLBM_READ_WRITE_ONLY) {
                g[q] = load_ro(base + (q * 64 + slot_of<TABLE>(q, x, y, z)));
                continue;
            }
            // q = 0 needs no test: its word is (own slot, delta 13), and bit
            // 0 of meta (the active bit) is set
            const uint32_t w = __ldg(&kPullTables[TABLE].w[q * 64 + j]);
            const int in_tile = (int)(w & 0x7ffu);
            const int bounced = (int)((w >> 11) & 0x7ffu);
            const bool link = (meta >> q) & 1u;
            if (REL32) {
                const int pulled = s_nbr[ti][w >> 22] + in_tile;
                g[q] = load_ro(base + (link ? pulled : bounced));
            } else {
                const T *src = link ? s_ptr[REL32 ? 0 : ti][w >> 22] : base;
                g[q] = load_ro(src + (link ? in_tile : bounced));
            }
        }

        if (VARIANT == TLBM_FULL) {
            const int tag = meta_type(meta);
            if (tag == BB_WALL) {
                // collision.py:250-252 reflect: f_new[q] = g[opp(q)]
#pragma unroll
                for (int q = 1; q < Q; ++q)
                    if (q < opp(q)) { T t = g[q]; g[q] = g[opp(q)]; g[opp(q)] = t; }
            } else {
                if (tag == INLET || tag == OUTLET)
                    zou_he<T, QUASI>(g, tag, meta_face(meta), p.inlet_u, p.outlet_rho);
                if constexpr (MRT && FMA)
                    status = collide_mrt_fma<T, QUASI>(g, p.mrt.op, T(p.guard_sq));
                else if constexpr (MRT)
                    status = collide_mrt<T, QUASI, TLBM_MRT_PACKED>(g, p.mrt.op, T(p.guard_sq),
                                                                    p.mrt.grouped);
                else if constexpr (FMA)
                    status = collide_fma<T, QUASI>(g, T(p.inv_tau), T(p.guard_sq));
                else
                    status = collide<T, QUASI>(g, T(p.inv_tau), T(p.guard_sq));
            }
        }
        T *out = p.dst + own;
#pragma unroll
        for (int q = 0; q < Q; ++q) store_out(out + (q * 64 + slot_of<TABLE>(q, x, y, z)), g[q]);
        if (HALO && p.halo_up && z == 3 && tile >= p.halo_up_begin &&
            tile < p.halo_up_end) {
            T *peer = p.halo_up + (tile - p.halo_up_begin) * TILE_VALUES;
#pragma unroll
            for (int k = 0; k < 5; ++k)
                peer[up_dir(k) * 64 + slot_of<TABLE>(up_dir(k), x, y, 3)] = g[up_dir(k)];
        }
        if (HALO && p.halo_down && z == 0 && tile >= p.halo_down_begin &&
            tile < p.halo_down_end) {
            T *peer = p.halo_down + (tile - p.halo_down_begin) * TILE_VALUES;
#pragma unroll
            for (int k = 0; k < 5; ++k)
                peer[opp(up_dir(k)) * 64 + slot_of<TABLE>(opp(up_dir(k)), x, y, 0)] =
                    g[opp(up_dir(k))];
        }
    }
    if (p.flags) {
        // one atomic per warp, and only for bits not yet set: a flow sitting at
        // the |u| guard must not serialise every warp on one L2 address
        const uint32_t any = __reduce_or_sync(0xffffffffu, status);
        if (any && (threadIdx.x & 31) == 0) {
            uint32_t *f = p.flags;
            if (p.iter)
                f += (unsigned long long)(*p.iter + p.iter_add) % p.ring_len;
            if (any & ~*reinterpret_cast<volatile uint32_t *>(f)) atomicOr(f, any);
        }
    }
}

}  // namespace step_detail
}  // namespace tlbm
#include "step_compact.cuh"
namespace tlbm {
namespace step_detail {

template <class T, int QUASI, int TABLE, int VARIANT, bool REL32, bool MRT, bool HALO, bool FMA>
int launch_as(const tlbm_step_args *a, cudaStream_t s);

template <class T, int QUASI, int TABLE, int VARIANT, bool MRT>
int launch_compact(const tlbm_step_args *a, cudaStream_t s);

template <class T, int QUASI, int TABLE, int VARIANT, bool REL32, bool MRT, bool FMA>
int launch_halo(const tlbm_step_args *a, cudaStream_t s) {
    if (VARIANT == TLBM_FULL && (a->halo_up || a->halo_down))
        return launch_as<T, QUASI, TABLE, VARIANT, REL32, MRT, VARIANT == TLBM_FULL, FMA>(a, s);
    return launch_as<T, QUASI, TABLE, VARIANT, REL32, MRT, false, FMA>(a, s);
}

inline bool mrt_moment_rates(const double *A, double *w);

// FMA arithmetic is fp64-only (tlbm_step rejects it for fp32).  An MRT
// operator that is not M^-1 diag(s) M (custom matrix) runs in reference
// arithmetic: bit-exact, so inside the FMA tolerance too.
inline bool fma_path(const tlbm_step_args *a, bool mrt) {
    double w[Q];
    return a->arith == TLBM_ARITH_FMA && (!mrt || mrt_moment_rates(a->mrt_op, w));
}

template <class T, int QUASI, int TABLE, int VARIANT, bool REL32, bool MRT>
int launch_arith(const tlbm_step_args *a, cudaStream_t s) {
    constexpr bool kFma = VARIANT == TLBM_FULL && sizeof(T) == 8;
    if (kFma && fma_path(a, MRT))
        return launch_halo<T, QUASI, TABLE, VARIANT, REL32, MRT, kFma>(a, s);
    return launch_halo<T, QUASI, TABLE, VARIANT, REL32, MRT, false>(a, s);
}

template <class T, int QUASI, int TABLE, int VARIANT>
int launch(const tlbm_step_args *a, cudaStream_t s) {
    if (a->crank) {
        if constexpr (compact_table_ok(TABLE)) {
            if (VARIANT == TLBM_FULL && a->collision == TLBM_MRT)
                return launch_compact<T, QUASI, TABLE, VARIANT, VARIANT == TLBM_FULL>(a, s);
            return launch_compact<T, QUASI, TABLE, VARIANT, false>(a, s);
        }
        set_error("tlbm_step: compact storage needs the xyz layout table");
        return TLBM_ERR_ARG;
    }
    if constexpr (VARIANT == TLBM_FULL) {     // MRT kernels only for the full step
        if (a->collision == TLBM_MRT) {
            if (a->rel32) return launch_arith<T, QUASI, TABLE, VARIANT, true, true>(a, s);
            return launch_arith<T, QUASI, TABLE, VARIANT, false, true>(a, s);
        }
    }
    if (a->rel32)
        return launch_arith<T, QUASI, TABLE, VARIANT, true, false>(a, s);
    return launch_arith<T, QUASI, TABLE, VARIANT, false, false>(a, s);
}

template <class T, bool MRT, bool FMA, int PACK>
void fill_params(StepParams<T, MRT> &p, const tlbm_step_args *a);

template <class T, int QUASI, int TABLE, int VARIANT, bool REL32, bool MRT, bool HALO, bool FMA>
int launch_as(const tlbm_step_args *a, cudaStream_t s) {
    StepParams<T, MRT> p;
    fill_params<T, MRT, FMA, TLBM_MRT_PACKED>(p, a);
    const long long n = a->tile_end - a->tile_begin;
    if (n <= 0) return TLBM_OK;
    constexpr int TPC = tiles_per_cta_of<T, MRT>();
    // the traversal order is a permutation of a whole-store launch; the
    // bench-ladder variants and the halo launches run in tile order
    if constexpr (VARIANT == TLBM_FULL && !HALO) {
        if (a->order) {
            step_kernel<T, QUASI, TABLE, VARIANT, TPC, REL32, MRT, HALO, FMA, true>
                <<<(unsigned)((n + TPC - 1) / TPC), 64 * TPC, 0, s>>>(p);
            return launch_check("step_kernel");
        }
    }
    step_kernel<T, QUASI, TABLE, VARIANT, TPC, REL32, MRT, HALO, FMA, false>
        <<<(unsigned)((n + TPC - 1) / TPC), 64 * TPC, 0, s>>>(p);
    return launch_check("step_kernel");
}

template <class T, int QUASI, int TABLE, int VARIANT, bool MRT, bool FMA>
int launch_nodes(const tlbm_step_args *a, cudaStream_t s) {
    StepParams<T, MRT> p;
    fill_params<T, MRT, FMA, TLBM_MRT_PACKED_COMPACT>(p, a);
    const long long n = a->node_end - a->node_begin;
    if (n <= 0) return TLBM_OK;
    constexpr int per_cta = TLBM_NODES_THREADS * nodes_per_thread<T, MRT>();
    const unsigned grid = (unsigned)((n + per_cta - 1) / per_cta);
    if (VARIANT == TLBM_FULL && (a->halo_up || a->halo_down))
        step_kernel_nodes<T, QUASI, TABLE, VARIANT, MRT, FMA, VARIANT == TLBM_FULL>
            <<<grid, TLBM_NODES_THREADS, 0, s>>>(p);
    else
        step_kernel_nodes<T, QUASI, TABLE, VARIANT, MRT, FMA, false>
            <<<grid, TLBM_NODES_THREADS, 0, s>>>(p);
    return launch_check("step_kernel_nodes");
}

template <class T, int QUASI, int TABLE, int VARIANT, bool MRT, bool FMA>
int launch_compact_as(const tlbm_step_args *a, cudaStream_t s) {
    StepParams<T, MRT> p;
    fill_params<T, MRT, FMA, TLBM_MRT_PACKED_COMPACT>(p, a);
    const long long n = a->tile_end - a->tile_begin;
    if (n <= 0) return TLBM_OK;
    constexpr int TPC = compact_tiles_per_cta<T>();
    const unsigned grid = (unsigned)((n + TPC - 1) / TPC);
    if constexpr (VARIANT == TLBM_FULL) {
        if (a->halo_up || a->halo_down) {
            if (a->rel32)
                step_kernel_compact<T, QUASI, TABLE, VARIANT, TPC, MRT, FMA, true, false, true>
                    <<<grid, 64 * TPC, 0, s>>>(p);
            else
                step_kernel_compact<T, QUASI, TABLE, VARIANT, TPC, MRT, FMA, false, false, true>
                    <<<grid, 64 * TPC, 0, s>>>(p);
            return launch_check("step_kernel_compact");
        }
        if (a->order) {
            if (a->rel32)
                step_kernel_compact<T, QUASI, TABLE, VARIANT, TPC, MRT, FMA, true, true, false>
                    <<<grid, 64 * TPC, 0, s>>>(p);
            else
                step_kernel_compact<T, QUASI, TABLE, VARIANT, TPC, MRT, FMA, false, true, false>
                    <<<grid, 64 * TPC, 0, s>>>(p);
            return launch_check("step_kernel_compact");
        }
    }
    if (a->rel32)       // for compact storage: 19 * n_fn < 2^32 (solver.py)
        step_kernel_compact<T, QUASI, TABLE, VARIANT, TPC, MRT, FMA, true, false, false>
            <<<grid, 64 * TPC, 0, s>>>(p);
    else
        step_kernel_compact<T, QUASI, TABLE, VARIANT, TPC, MRT, FMA, false, false, false>
            <<<grid, 64 * TPC, 0, s>>>(p);
    return launch_check("step_kernel_compact");
}

template <class T, int QUASI, int TABLE, int VARIANT, bool MRT>
int launch_compact(const tlbm_step_args *a, cudaStream_t s) {
    const bool halo = a->halo_up || a->halo_down;
    if (halo && (VARIANT != TLBM_FULL || a->order ||
                 (a->halo_up && !a->halo_up_cbase) || (a->halo_down && !a->halo_down_cbase))) {
        set_error("tlbm_step: the compact fused halo needs the full step in tile order and "
                  "the neighbours' ghost block offsets (halo_*_cbase)");
        return TLBM_ERR_ARG;
    }
    if (!a->cbase || !a->cnf) {
        set_error("tlbm_step: compact storage needs cbase, cnf and crank");
        return TLBM_ERR_ARG;
    }
    constexpr bool kFma = VARIANT == TLBM_FULL && sizeof(T) == 8;
    if (a->node_meta) {
        if (!a->node_rec || !a->unit_tile || !a->entries || !a->rel32 || a->order ||
            a->node_begin < 0 || a->node_end < a->node_begin) {
            set_error("tlbm_step: the node-parallel step needs node_rec, unit_tile, entries, "
                      "a node range, 32-bit offsets (rel32) and tile order");
            return TLBM_ERR_ARG;
        }
        if (kFma && fma_path(a, MRT)) return launch_nodes<T, QUASI, TABLE, VARIANT, MRT, kFma>(a, s);
        return launch_nodes<T, QUASI, TABLE, VARIANT, MRT, false>(a, s);
    }
    if (kFma && fma_path(a, MRT))
        return launch_compact_as<T, QUASI, TABLE, VARIANT, MRT, kFma>(a, s);
    return launch_compact_as<T, QUASI, TABLE, VARIANT, MRT, false>(a, s);
}

// Is A = M^-1 diag(s) M in the collision.py moment basis, with s = 0 on the
// conserved moments?  B = M A M^T D^-1 must be diagonal to 1e-12 of its
// largest entry; then w[k] = s_k / |M_k|^2 (FMA-arithmetic moment path).
inline bool mrt_moment_rates_uncached(const double *A, double *w) {
    double MA[Q][Q];
    for (int k = 0; k < Q; ++k)
        for (int r = 0; r < Q; ++r) {
            double acc = 0.0;
            for (int q = 0; q < Q; ++q) acc += moment_coef(k, q) * A[q * Q + r];
            MA[k][r] = acc;
        }
    double B[Q][Q], big = 0.0;
    for (int k = 0; k < Q; ++k)
        for (int l = 0; l < Q; ++l) {
            double acc = 0.0;
            for (int r = 0; r < Q; ++r) acc += MA[k][r] * moment_coef(l, r);
            B[k][l] = acc / moment_norm(l);
            big = std::max(big, std::fabs(B[k][l]));
        }
    const double tol = 1e-12 * std::max(big, 1.0);
    for (int k = 0; k < Q; ++k) {
        for (int l = 0; l < Q; ++l)
            if (l != k && !(std::fabs(B[k][l]) <= tol)) return false;
        if (moment_conserved(k) && !(std::fabs(B[k][k]) <= tol)) return false;
        w[k] = moment_conserved(k) ? 0.0 : B[k][k] / moment_norm(k);
    }
    return true;
}

inline bool mrt_moment_rates(const double *A, double *w) {
    // per-thread memo of the last operator (fill_params runs every launch)
    thread_local double last_A[Q * Q], last_w[Q];
    thread_local bool last_ok = false, have = false;
    if (have && memcmp(last_A, A, sizeof(last_A)) == 0) {
        memcpy(w, last_w, sizeof(last_w));
        return last_ok;
    }
    have = false;
    memcpy(last_A, A, sizeof(last_A));
    last_ok = mrt_moment_rates_uncached(A, last_w);
    have = true;
    memcpy(w, last_w, sizeof(last_w));
    return last_ok;
}

template <class T, bool MRT, bool FMA, int PACK>
void fill_params(StepParams<T, MRT> &p, const tlbm_step_args *a) {
    if constexpr (MRT) {
        // op.astype(dtype); grouped when every column's equal-value rows of
        // the compiled pattern hold bitwise-equal coefficients; in FMA
        // arithmetic, moment space when op = M^-1 diag(s) M
        double w[Q];
        if (FMA && !mrt_moment_rates(a->mrt_op, w))   // launch_arith routes these
            for (int k = 0; k < Q; ++k) w[k] = 0.0;   // to reference arithmetic
        bool grouped = !FMA && TLBM_MRT_GROUPED;
        for (int i = 0; i < Q && grouped; ++i)
            for (int j = 0; j < Q && grouped; ++j) {
                const T c = T(a->mrt_op[i * Q + j]);
                const T rep = T(a->mrt_op[mrt_rep(mrt_offset(j) + mrt_group(i, j)) * Q + j]);
                grouped = memcmp(&c, &rep, sizeof(T)) == 0;
            }
        p.mrt.grouped = grouped;
        if (FMA)
            for (int k = 0; k < Q; ++k) p.mrt.op[k] = T(w[k]);
        else if (grouped && sizeof(T) == 4 && PACK == 2) {
            // (c_a, c_b) per combination, then the single row's scalars
            auto val = [&](int j, int k) { return T(a->mrt_op[mrt_rep(mrt_offset(j) + k) * Q + j]); };
            for (int j = 0; j < Q; ++j) {
                for (int c = 0; c < mrt_ncombo(j); ++c)
                    for (int h = 0; h < 2; ++h)
                        p.mrt.op[2 * (mrt_combo_offset(j) + c) + h] = val(j, mrt_combo_group(j, c, h));
                if (mrt_single_offset(j) >= 0)
                    p.mrt.op[mrt_single_offset(j)] = val(j, mrt_group(kMrtSingleRow, j));
            }
        } else if (grouped)
            for (int j = 0; j < Q; ++j)
                for (int k = 0; k < mrt_count(j); ++k)
                    p.mrt.op[mrt_table_offset<T, PACK>(j) + k] =
                        T(a->mrt_op[mrt_rep(mrt_offset(j) + k) * Q + j]);
        else
            for (int k = 0; k < Q * Q; ++k) p.mrt.op[k] = T(a->mrt_op[k]);
    }
    p.src = static_cast<const T *>(a->f_src);
    p.dst = static_cast<T *>(a->f_dst);
    p.nbr = a->nbr;
    p.meta = a->meta;
    p.tile_begin = a->tile_begin;
    p.tile_end = a->tile_end;
    p.inv_tau = 1.0 / a->tau;
    for (int k = 0; k < 3; ++k) p.inlet_u[k] = a->inlet_u[k];
    p.outlet_rho = a->outlet_rho;
    p.guard_sq = a->u_guard > 0.0 ? a->u_guard * a->u_guard : HUGE_VAL;
    p.flags = a->flags;
    p.iter = reinterpret_cast<const long long *>(a->iter_counter);
    p.iter_add = a->iter_add;
    p.ring_len = (unsigned long long)(a->ring_len > 0 ? a->ring_len : 1);
    p.halo_up = static_cast<T *>(a->halo_up);
    p.halo_up_begin = a->halo_up_begin;
    p.halo_up_end = a->halo_up_end;
    p.halo_down = static_cast<T *>(a->halo_down);
    p.halo_down_begin = a->halo_down_begin;
    p.halo_down_end = a->halo_down_end;
    p.cbase = reinterpret_cast<const long long *>(a->cbase);
    p.cnf = a->cnf;
    p.crank = a->crank;
    p.order = a->order;
    p.halo_up_cbase = reinterpret_cast<const long long *>(a->halo_up_cbase);
    p.halo_down_cbase = reinterpret_cast<const long long *>(a->halo_down_cbase);
    p.node_meta = a->node_meta;
    p.node_rec = a->node_rec;
    p.unit_tile = a->unit_tile;
    p.entries = a->entries;
    p.node_begin = a->node_begin;
    p.node_end = a->node_end;
    p.scale_value = sizeof(T);
    p.scale_entry = sizeof(uint2);
}

template <class T>
struct StepLaunch {
    const tlbm_step_args *a;
    cudaStream_t s;
    template <int QUASI, int TABLE>
    int run() const {
        switch (a->variant) {
            case TLBM_FULL: return launch<T, QUASI, TABLE, TLBM_FULL>(a, s);
            case TLBM_PROPAGATION_ONLY:
                return QUASI ? TLBM_OK : launch<T, 0, TABLE, TLBM_PROPAGATION_ONLY>(a, s);
            case TLBM_READ_WRITE_ONLY:
                return QUASI ? TLBM_OK : launch<T, 0, TABLE, TLBM_READ_WRITE_ONLY>(a, s);
        }
        set_error("unknown step variant %d", a->variant);
        return TLBM_ERR_ARG;
    }
};

// one translation unit per dtype (step_f64.cu / step_f32.cu) instantiates
// this, so the 72 (fp32) and 120 (fp64) kernels compile in parallel
template <class T>
int launch_dtype(const tlbm_step_args *a, cudaStream_t s) {
    const StepLaunch<T> l{a, s};
    const int fluid = (a->variant == TLBM_FULL) ? a->fluid : TLBM_INCOMPRESSIBLE;
#define TLBM_T(QU, TB) \
    if (fluid == QU && a->table == TB) return l.template run<QU, TB>();
    TLBM_T(0, 0) TLBM_T(0, 1) TLBM_T(0, 2) TLBM_T(1, 0) TLBM_T(1, 1) TLBM_T(1, 2)
#undef TLBM_T
    set_error("tlbm_step: bad fluid %d / table %d", fluid, a->table);
    return TLBM_ERR_ARG;
}

}  // namespace step_detail
}  // namespace tlbm
