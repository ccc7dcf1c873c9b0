// The fused step on the compact tile store (compact.cu): the same pull
// gather, boundary handling, collision and store as step_kernel
// (step_impl.cuh), with every block holding only its tile's non-solid slots.
//
// Why: on a sparse geometry the paper's 64-slot blocks put solid slots next
// to fluid ones, so DRAM moves whole 32-byte sectors of which part is never
// used, and partially written sectors cost a fill read.  Packing the blocks
// removes both: scripts/sparse_traffic_model.py gives 152 B read + 152 B
// written per fluid node at every porosity (fp64), against 177 + 177 B plus
// 1.5 partial sectors per node at porosity 0.2 in the paper's layout.
//
// In-block order: the compact store keeps every block in the canonical
// (XYZ) slot order, so a node's rank -- its index among its tile's non-solid
// slots -- is the same in all 19 blocks of the tile.  The per-layout sector
// tricks of the B200 table do not apply once blocks are packed; packing is
// what removes the over-fetch.
//
// Addressing per pull (direction q, packed word w of the XYZ pull table):
//   link:    source tile k = neighbour row entry w >> 22, slot s = w & 63,
//            block q
//   no link: own tile, the node's own slot, block opp(q)
//   addr = base(k) + block * nf(k) + rank(k, s)
// The CTA stages base/nf and the 64 one-byte ranks (crank, built at setup)
// of the 27 neighbour tiles in shared memory, so a pull's rank is one byte
// load from shared memory.
#pragma once

namespace tlbm {
namespace step_detail {

// occupancy of the compact kernel (resident warps per SM): fp64 32 (64
// registers); fp32 48 (40 registers, no spills with OFF32 addressing;
// measured 23.4 / 28.0 / 32.5 GLUPS at porosity 0.2 / 0.5 / 1.0 vs 21.3 /
// 25.6 / 28.0 at 32 warps, and the same at 64 warps with an 8-byte spill)
#ifndef TLBM_WARPS_COMPACT
#define TLBM_WARPS_COMPACT 32
#endif
#ifndef TLBM_WARPS_COMPACT_F32
#define TLBM_WARPS_COMPACT_F32 48
#endif
#ifndef TLBM_WARPS_NODES_F32
#define TLBM_WARPS_NODES_F32 (TLBM_NODES_NPT_F32 == 1 ? 48 : TLBM_NODES_NPT_F32 == 2 ? 32 : 24)
#endif
// per (q, j): 64 * (neighbour-row entry of the source tile) + source slot
struct CompactPull {
    uint16_t w[Q * 64];
};
constexpr CompactPull make_compact_pull() {
    CompactPull t{};
    for (int q = 0; q < Q; ++q)
        for (int j = 0; j < 64; ++j) {
            const int x = j & 3, y = (j >> 2) & 3, z = j >> 4;
            const int sx = x - ex(q), sy = y - ey(q), sz = z - ez(q);
            const int dx = sx < 0 ? -1 : (sx > 3 ? 1 : 0);
            const int dy = sy < 0 ? -1 : (sy > 3 ? 1 : 0);
            const int dz = sz < 0 ? -1 : (sz > 3 ? 1 : 0);
            t.w[q * 64 + j] = (uint16_t)(64 * delta_index(dx, dy, dz) +
                                         ((sx & 3) + 4 * (sy & 3) + 16 * (sz & 3)));
        }
    return t;
}
__device__ const CompactPull kCompactPull = make_compact_pull();

#ifndef TLBM_TPC_COMPACT
#define TLBM_TPC_COMPACT 2
#endif
template <class T>
constexpr int compact_tiles_per_cta() { return sizeof(T) == 4 ? 1 : TLBM_TPC_COMPACT; }

template <class T, bool MRT, int VARIANT, bool FMA = false>
constexpr int min_blocks_compact() {
    return (MRT ? (sizeof(T) == 4 ? TLBM_WARPS_COMPACT_MRT_F32
                                  : (FMA ? TLBM_WARPS_MRT_FMA : TLBM_WARPS_MRT))
                : (sizeof(T) == 4 ? TLBM_WARPS_COMPACT_F32 : TLBM_WARPS_COMPACT)) /
           (2 * compact_tiles_per_cta<T>());
}

// element i of base, scale = sizeof(T) passed at run time (StepParams::
// scale_*) so the address is one IMAD.WIDE.U32 on the FMA pipe
template <class T>
__device__ __forceinline__ T *at_u32(T *base, unsigned i, unsigned scale) {
    using B = std::conditional_t<std::is_const_v<T>, const char, char>;
    return reinterpret_cast<T *>(reinterpret_cast<B *>(base) + (unsigned long long)i * scale);
}

// The tail of a node's update on the compact store, shared by the compact
// kernels: boundary handling, collision, the store into the other copy at
// own + q * nf_own + rank_own, and the fused halo.
template <class T, int QUASI, int VARIANT, bool MRT, bool FMA, bool HALO, class Off>
__device__ __forceinline__ uint32_t compact_finish(const StepParams<T, MRT> &p, long long tile,
                                                   int j, uint32_t meta, T (&g)[Q], Off own,
                                                   int nf_own, int rank_own) {
    uint32_t status = 0;
    if (VARIANT == TLBM_FULL) {
        const int tag = meta_type(meta);
        if (tag == BB_WALL) {
#pragma unroll
            for (int q = 1; q < Q; ++q)
                if (q < opp(q)) { T t = g[q]; g[q] = g[opp(q)]; g[opp(q)] = t; }
        } else {
            if (tag == INLET || tag == OUTLET)
                zou_he<T, QUASI>(g, tag, meta_face(meta), p.inlet_u, p.outlet_rho);
            if constexpr (MRT && FMA)
                status = collide_mrt_fma<T, QUASI>(g, p.mrt.op, T(p.guard_sq));
            else if constexpr (MRT)
                status = collide_mrt<T, QUASI, TLBM_MRT_PACKED_COMPACT>(g, p.mrt.op, T(p.guard_sq),
                                                                        p.mrt.grouped);
            else if constexpr (FMA)
                status = collide_fma<T, QUASI>(g, T(p.inv_tau), T(p.guard_sq));
            else
                status = collide<T, QUASI>(g, T(p.inv_tau), T(p.guard_sq));
        }
    }
    if constexpr (std::is_same_v<Off, unsigned>) {
        // 32-bit offsets: one IMAD + one IMAD.WIDE per store
        T *out = at_u32(p.dst, own + (unsigned)rank_own, p.scale_value);
#pragma unroll
        for (int q = 0; q < Q; ++q)
            store_out(at_u32(out, (unsigned)(q * nf_own), p.scale_value), g[q]);
    } else {
        T *out = p.dst + own;
#pragma unroll
        for (int q = 0; q < Q; ++q) store_out(out + (q * nf_own + rank_own), g[q]);
    }
    if constexpr (HALO) {
        // fused halo: the neighbour's ghost copy of this tile has the same
        // nodes (same ranks and count), at its own block offset
        const int z = j >> 4;
        if (p.halo_up && z == 3 && tile >= p.halo_up_begin && tile < p.halo_up_end) {
            T *peer = p.halo_up + p.halo_up_cbase[tile - p.halo_up_begin];
#pragma unroll
            for (int k = 0; k < 5; ++k)
                peer[up_dir(k) * nf_own + rank_own] = g[up_dir(k)];
        }
        if (p.halo_down && z == 0 && tile >= p.halo_down_begin && tile < p.halo_down_end) {
            T *peer = p.halo_down + p.halo_down_cbase[tile - p.halo_down_begin];
#pragma unroll
            for (int k = 0; k < 5; ++k)
                peer[opp(up_dir(k)) * nf_own + rank_own] = g[opp(up_dir(k))];
        }
    }
    return status;
}

// a neighbour entry as the update sees it: block offset (unsigned 32-bit
// from the copy start, or 64-bit) and block length
template <class Off>
struct Entry {
    Off off;
    int nf;
};

// One node's update in the tile-parallel compact kernel: pull gather
// through the staged neighbourhood (rank bytes rank[k * 64 + s] and
// entry(k) = block offset and length of the 27 neighbour entries, entry 13 =
// the node's own tile), then compact_finish.  The offset is an unsigned
// 32-bit element offset from the copy start (OFF32) or a 64-bit one.
template <class T, int QUASI, int VARIANT, bool MRT, bool FMA, bool HALO, class E>
__device__ __forceinline__ uint32_t compact_update(const StepParams<T, MRT> &p, long long tile,
                                                   int j, uint32_t meta,
                                                   const unsigned char *rank, E entry) {
    const T *base0 = opaque(p.src);
    const auto mine = entry(13);
    const auto own = mine.off;
    const int nf_own = mine.nf;
    const int rank_own = rank[13 * 64 + j];
    T g[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (VARIANT == TLBM_READ_WRITE_ONLY || q == 0) {
            g[q] = load_ro(base0 + (own + (decltype(own))(q * nf_own + rank_own)));
            continue;
        }
        // w = 64 * (source tile entry) + source slot
        const uint32_t w = __ldg(&kCompactPull.w[q * 64 + j]);
        const bool link = (meta >> q) & 1u;
        const int k = link ? (int)(w >> 6) : 13;
        const int r = link ? (int)rank[w] : rank_own;
        const int blk = link ? q : opp(q);
        const auto e = entry(k);
        g[q] = load_ro(base0 + (e.off + (decltype(own))(blk * e.nf + r)));
    }
    return compact_finish<T, QUASI, VARIANT, MRT, FMA, HALO>(p, tile, j, meta, g, own, nf_own,
                                                             rank_own);
}

// OR a warp's status bits into the launch's status word (one conditional
// atomic per warp; see step_kernel)
template <class P>
__device__ __forceinline__ void report_status(const P &p, uint32_t status) {
    if (p.flags) {
        const uint32_t any = __reduce_or_sync(0xffffffffu, status);
        if (any && (threadIdx.x & 31) == 0) {
            uint32_t *f = p.flags;
            if (p.iter)
                f += (unsigned long long)(*p.iter + p.iter_add) % p.ring_len;
            if (any & ~*reinterpret_cast<volatile uint32_t *>(f)) atomicOr(f, any);
        }
    }
}

// no D3Q19 pull reads one of the 8 corner neighbours: they are not staged
__host__ __device__ constexpr bool corner_entry(int k) {
    return k == 0 || k == 2 || k == 6 || k == 8 || k == 18 || k == 20 || k == 24 || k == 26;
}

// OFF32: every element offset of a copy fits 32 bits (19 * n_fn < 2^32, i.e.
// up to 226 M fluid nodes): neighbour block starts are staged as 32-bit
// offsets from the copy start and each pull is one 32-bit add chain plus one
// IMAD.WIDE.U32 from a single base -- fewer live registers than a 64-bit
// offset per pull.
template <class T, int QUASI, int TABLE, int VARIANT, int TPC, bool MRT, bool FMA, bool OFF32,
          bool ORDERED, bool HALO>
__global__ void __launch_bounds__(64 * TPC, min_blocks_compact<T, MRT, VARIANT, FMA>())
step_kernel_compact(const StepParams<T, MRT> p) {
    static_assert(compact_table_ok(TABLE), "compact storage keeps blocks in XYZ order");
    __shared__ long long s_src[OFF32 ? 1 : TPC][NBR];
    __shared__ unsigned s_off[OFF32 ? TPC : 1][NBR];
    __shared__ int s_nf[TPC][NBR];
    __shared__ __align__(16) unsigned char s_rank[TPC][NBR][64];
    const int ti = threadIdx.x >> 6;
    const int j = threadIdx.x & 63;
    const long long pos0 = p.tile_begin + (long long)blockIdx.x * TPC;
    const bool valid = pos0 + ti < p.tile_end;
    const long long tile = valid ? tile_at<ORDERED>(p, pos0 + ti) : 0;

    // the node word does not depend on the staging: load it first so its
    // latency overlaps the neighbour rows
    const uint32_t meta = valid ? p.meta[tile * 64 + j] : 0u;
    // neighbour rows, then each neighbour's 64 ranks as four 16-byte copies
    for (int i = threadIdx.x; i < TPC * NBR; i += 64 * TPC) {
        const bool ok = pos0 + i / NBR < p.tile_end;
        const long long t = ok ? tile_at<ORDERED>(p, pos0 + i / NBR) : 0;
        const int k = i % NBR;
        if (corner_entry(k)) continue;
        long long nb = -1;
        if (ok) nb = VARIANT == TLBM_READ_WRITE_ONLY ? (k == 13 ? t : -1) : p.nbr[t * NBR + k];
        const long long tt = nb >= 0 ? nb : t;
        if (OFF32) s_off[OFF32 ? i / NBR : 0][k] = (unsigned)p.cbase[tt];
        else s_src[OFF32 ? 0 : i / NBR][k] = p.cbase[tt];
        s_nf[i / NBR][k] = p.cnf[tt];
        const uint4 *r = reinterpret_cast<const uint4 *>(p.crank + tt * 64);
        uint4 *d = reinterpret_cast<uint4 *>(&s_rank[i / NBR][k][0]);
#pragma unroll
        for (int c = 0; c < 4; ++c) d[c] = __ldg(r + c);
    }
    __syncthreads();

    uint32_t status = 0;
    if (meta & META_ACTIVE) {
        if constexpr (OFF32)
            status = compact_update<T, QUASI, VARIANT, MRT, FMA, HALO>(
                p, tile, j, meta, &s_rank[ti][0][0],
                [&](int k) { return Entry<unsigned>{s_off[ti][k], s_nf[ti][k]}; });
        else
            status = compact_update<T, QUASI, VARIANT, MRT, FMA, HALO>(
                p, tile, j, meta, &s_rank[ti][0][0],
                [&](int k) { return Entry<long long>{s_src[ti][k], s_nf[ti][k]}; });
    }
    report_status(p, status);
}

// ---- node-parallel compact step -------------------------------------------
// One thread per non-solid node, in store order, so the lanes a partly solid
// tile leaves idle in the tile-parallel kernel (a third at porosity 0.2) do
// work.  Each node's pull sources come from its precomputed record
// (tlbm_compact_nodes): the 18 source ranks, its own rank and its tile; the
// source tile's block offset and length come from the tile's 27-entry row of
// {offset, count} (8-byte loads that the lanes of one tile share in L1);
// which entry a pull reads follows from the slot by integer arithmetic, so
// the gather sits three load levels deep (record -> entry -> value).  Node-level
// metadata is 20 B + 216 B per tile (~25 B per fluid node at porosity 0.2,
// 8% of the 304 B the populations move in fp64).
#ifndef TLBM_NODES_THREADS
#define TLBM_NODES_THREADS 128
#endif
// nodes per thread of the fp32 LBGK node-parallel step: two, at 32 warps/SM
// (64 registers), beat one at 48 warps/SM by 2-3% below porosity 0.6
// (scripts/exp/exp50.sh)
#ifndef TLBM_NODES_NPT_F32
#define TLBM_NODES_NPT_F32 2
#endif
#ifndef TLBM_NODES_NPT_F64
#define TLBM_NODES_NPT_F64 1
#endif
#ifndef TLBM_WARPS_NODES_F64
#define TLBM_WARPS_NODES_F64 (TLBM_NODES_NPT_F64 == 1 ? TLBM_WARPS_COMPACT : 16)
#endif
template <class T, bool MRT>
constexpr int nodes_per_thread() {
    return MRT ? 1 : (sizeof(T) == 4 ? TLBM_NODES_NPT_F32 : TLBM_NODES_NPT_F64);
}
template <class T, bool MRT, bool FMA = false>
constexpr int min_blocks_nodes() {
    return (MRT ? (sizeof(T) == 4 ? TLBM_WARPS_COMPACT_MRT_F32
                                  : (FMA ? TLBM_WARPS_MRT_FMA : TLBM_WARPS_MRT))
                : (sizeof(T) == 4 ? TLBM_WARPS_NODES_F32 : TLBM_WARPS_NODES_F64)) /
           (TLBM_NODES_THREADS / 32);
}

// what the tail of a node's update needs besides its gathered values
struct NodeCtx {
    long long tile;
    uint32_t meta;
    unsigned own;
    int nf_own, rank_own;
};

// one node's gather; rec / meta / unit_tile already loaded
template <class T, int VARIANT, bool MRT>
__device__ __forceinline__ NodeCtx node_gather(const StepParams<T, MRT> &p, uint32_t meta,
                                               uint4 rec, int unit_tile, T (&g)[Q]) {
    const int j = (int)(meta >> 25);
    const int rank_own = (int)((rec.w >> 18) & 63u);
    const long long tile = (long long)unit_tile + ((rec.w >> 24) & 63u);
    const uint2 *ent = reinterpret_cast<const uint2 *>(p.entries) + tile * NBR;
    const uint2 mine = __ldg(ent + 13);
    const unsigned own = mine.x;
    const int nf_own = (int)mine.y;
    const T *base0 = p.src;
    // neighbour-row entry of each pull without a table load: a pull in
    // direction e crosses into the tile at -e on the axes where the slot
    // sits on the face it pulls across; the entry index is 13 plus the
    // crossing axes' contributions (9, 3, 1 per tile step in x, y, z)
    const int x = j & 3, y = (j >> 2) & 3, z = j >> 4;
    const int cx[2] = {x == 0 ? -9 : 0, x == 3 ? 9 : 0};   // e_x = +1, -1
    const int cy[2] = {y == 0 ? -3 : 0, y == 3 ? 3 : 0};
    const int cz[2] = {z == 0 ? -1 : 0, z == 3 ? 1 : 0};
    const unsigned own_r = own + (unsigned)rank_own;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (VARIANT == TLBM_READ_WRITE_ONLY || q == 0) {
            g[q] = load_ro(at_u32(base0, own + (unsigned)(q * nf_own + rank_own), p.scale_value));
            continue;
        }
        // the record holds the source rank (the node's own rank where there
        // is no link; halfway bounce-back reads block opp(q) of its own tile)
        const uint32_t word = (q - 1) < 5 ? rec.x : (q - 1) < 10 ? rec.y
                            : (q - 1) < 15 ? rec.z : rec.w;
        const int r = (int)((word >> (6 * ((q - 1) % 5))) & 63u);
        // the entry of the pull's source tile is read whether or not the
        // link exists (every entry is valid: a missing neighbour is the tile
        // itself), so only the final offset is selected
        const bool link = (meta >> q) & 1u;
        const int kq = 13 + (ex(q) > 0 ? cx[0] : ex(q) < 0 ? cx[1] : 0) +
                       (ey(q) > 0 ? cy[0] : ey(q) < 0 ? cy[1] : 0) +
                       (ez(q) > 0 ? cz[0] : ez(q) < 0 ? cz[1] : 0);
        const uint2 e = __ldg(at_u32(ent, (unsigned)kq, p.scale_entry));
        const unsigned pulled = e.x + (unsigned)(q * (int)e.y + r);
        const unsigned bounced = own_r + (unsigned)(opp(q) * nf_own);
        g[q] = load_ro(at_u32(base0, link ? pulled : bounced, p.scale_value));
    }
    return NodeCtx{tile, meta, own, nf_own, rank_own};
}

template <class T, int QUASI, int VARIANT, bool MRT, bool FMA, bool HALO>
__device__ __forceinline__ uint32_t node_finish(const StepParams<T, MRT> &p, const NodeCtx &c,
                                                T (&g)[Q]) {
    return compact_finish<T, QUASI, VARIANT, MRT, FMA, HALO>(
        p, c.tile, (int)(c.meta >> 25), c.meta, g, c.own, c.nf_own, c.rank_own);
}

template <class T, int VARIANT, bool MRT>
__device__ __forceinline__ NodeCtx node_load_gather(const StepParams<T, MRT> &p, long long n,
                                                    T (&g)[Q]) {
    return node_gather<T, VARIANT, MRT>(
        p, __ldg(p.node_meta + n), __ldg(reinterpret_cast<const uint4 *>(p.node_rec) + n),
        __ldg(p.unit_tile + (n >> 6)), g);
}

template <class T, int QUASI, int TABLE, int VARIANT, bool MRT, bool FMA, bool HALO>
__global__ void __launch_bounds__(TLBM_NODES_THREADS, min_blocks_nodes<T, MRT, FMA>())
step_kernel_nodes(const StepParams<T, MRT> p) {
    static_assert(compact_table_ok(TABLE), "compact storage keeps blocks in XYZ order");
    constexpr int NPT = nodes_per_thread<T, MRT>();
    uint32_t status = 0;
    const long long n = p.node_begin + (long long)blockIdx.x * TLBM_NODES_THREADS * NPT +
                        threadIdx.x;
    if constexpr (NPT == 1) {
        if (n < p.node_end) {
            T g[Q];
            const NodeCtx c = node_load_gather<T, VARIANT, MRT>(p, n, g);
            status = node_finish<T, QUASI, VARIANT, MRT, FMA, HALO>(p, c, g);
        }
    } else {
        // NPT nodes per thread, CTA-strided: every gather in flight before
        // the first update (a node past the end gathers the last node again
        // and is not stored)
        if (n < p.node_end) {
            T g[NPT][Q];
            NodeCtx c[NPT];
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const long long nk = n + (long long)k * TLBM_NODES_THREADS;
                c[k] = node_load_gather<T, VARIANT, MRT>(p, nk < p.node_end ? nk : p.node_end - 1,
                                                         g[k]);
            }
#pragma unroll
            for (int k = 0; k < NPT; ++k)
                if (k == 0 || n + (long long)k * TLBM_NODES_THREADS < p.node_end)
                    status |= node_finish<T, QUASI, VARIANT, MRT, FMA, HALO>(p, c[k], g[k]);
        }
    }
    report_status(p, status);
}

}  // namespace step_detail
}  // namespace tlbm
