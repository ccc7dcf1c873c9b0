// Compact tile storage (an extension of the paper's layout):
// the field store keeps only the non-solid slots of every (tile, direction)
// block, in the canonical (XYZ) slot order.  Tile T's 19 blocks start at
// base(T) = 19 * (non-solid nodes of the tiles before T); block q is nf(T)
// values long; the node at canonical slot j sits at its rank among T's
// non-solid slots, the same in all 19 blocks:
//     addr(T, q, j) = base(T) + q * nf(T) + rank(T, j)
// A block of the paper's XYZ layout is the same values with the solid slots
// left in place.
//
// This file: the per-tile rank bytes and the conversion between the paper's
// block store ([tile][q][64], layout.py:115-132) and the compact one, which
// is how every canonical read/write (init, readout, checkpoints) reaches a
// compact store.  The compact step kernel is in step_compact.cuh.
#include "common.cuh"
#include "d3q19.cuh"

namespace tlbm {
namespace {

constexpr int TILE_VALUES = Q * 64;

// rank[t][j] = number of non-solid slots of tile t before slot j (255 for a
// solid slot); one warp per tile, a ballot gives the tile's 64-bit mask
__global__ void ranks_kernel(const uint32_t *meta, long long t_n, unsigned char *rank) {
    const long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= t_n) return;
    const bool a0 = meta[t * 64 + lane] & META_ACTIVE;
    const bool a1 = meta[t * 64 + 32 + lane] & META_ACTIVE;
    const unsigned lo = __ballot_sync(0xffffffffu, a0), hi = __ballot_sync(0xffffffffu, a1);
    const unsigned below = (1u << lane) - 1u;
    rank[t * 64 + lane] = a0 ? (unsigned char)__popc(lo & below) : 255;
    rank[t * 64 + 32 + lane] = a1 ? (unsigned char)(__popc(lo) + __popc(hi & below)) : 255;
}

template <class T, bool TO_COMPACT>
__global__ void convert_kernel(const T *in, T *out, long long t_n, const long long *base,
                               const int *nf, const unsigned char *rank) {
    const long long n = t_n * 64;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long t = i >> 6;
        const int j = (int)(i & 63);
        const int r = rank[i];
        if (r == 255) {
            if (!TO_COMPACT) {
                // solid slots do not exist in a compact store; expand them as
                // the rest state w_q (rho 1, u 0), what a never-written slot
                // of the paper's store holds after the cold start
#pragma unroll
                for (int q = 0; q < Q; ++q) out[t * TILE_VALUES + q * 64 + j] = T(weight(q));
            }
            continue;
        }
        const long long b = base[t] + r;
        const int n_t = nf[t];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const long long c = b + (long long)q * n_t;
            const long long f = t * TILE_VALUES + q * 64 + j;
            if (TO_COMPACT) out[c] = in[f];
            else out[f] = in[c];
        }
    }
}

unsigned grid_for_slots(long long n) {
    long long g = (n + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148LL * 32) g = 148LL * 32;
    return (unsigned)g;
}

template <class T>
int convert_as(const void *in, void *out, int64_t t_n, const int64_t *base, const int32_t *nf,
               const uint8_t *rank, int to_compact, cudaStream_t s) {
    const auto *b = reinterpret_cast<const long long *>(base);
    if (to_compact)
        convert_kernel<T, true><<<grid_for_slots(t_n * 64), 256, 0, s>>>(
            static_cast<const T *>(in), static_cast<T *>(out), t_n, b, nf, rank);
    else
        convert_kernel<T, false><<<grid_for_slots(t_n * 64), 256, 0, s>>>(
            static_cast<const T *>(in), static_cast<T *>(out), t_n, b, nf, rank);
    return launch_check("convert_kernel");
}

}  // namespace
}  // namespace tlbm

using namespace tlbm;

extern "C" int tlbm_compact_ranks(const uint32_t *d_meta, int64_t t_n, uint8_t *d_rank,
                                  void *stream) {
    if (t_n == 0) return TLBM_OK;             // no tiles: nothing to rank
    if (!d_meta || !d_rank || t_n < 0) {
        set_error("tlbm_compact_ranks: bad argument");
        return TLBM_ERR_ARG;
    }
    ranks_kernel<<<(unsigned)((t_n * 32 + 255) / 256), 256, 0, as_stream(stream)>>>(
        d_meta, (long long)t_n, d_rank);
    return launch_check("ranks_kernel");
}

extern "C" int tlbm_compact_convert(const void *d_in, void *d_out, int dtype, int table,
                                    int64_t t_n, const int64_t *d_base, const int32_t *d_nf,
                                    const uint8_t *d_rank, int to_compact, void *stream) {
    int rc;
    if ((rc = check_dtype(dtype)) || (rc = check_table(table))) return rc;
    if (!compact_table_ok(table)) {
        set_error("compact storage keeps blocks in XYZ order: needs the xyz table, got %d",
                  table);
        return TLBM_ERR_ARG;
    }
    if (t_n == 0) return TLBM_OK;
    if (!d_in || !d_out || !d_base || !d_nf || !d_rank) {
        set_error("tlbm_compact_convert: null argument");
        return TLBM_ERR_ARG;
    }
    cudaStream_t s = as_stream(stream);
    return dtype == TLBM_F64 ? convert_as<double>(d_in, d_out, t_n, d_base, d_nf, d_rank,
                                                  to_compact, s)
                             : convert_as<float>(d_in, d_out, t_n, d_base, d_nf, d_rank,
                                                 to_compact, s);
}

// ---- per-node records for the node-parallel step ---------------------------
// (layout in include/tlbm.h: tlbm_compact_nodes; kernel step_kernel_nodes)
namespace tlbm {
namespace {

// the tile of node 64u, for every unit u that starts inside tile t
__global__ void unit_tile_kernel(const long long *base, const int *nf, long long t_n,
                                 int *unit_tile) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < t_n;
         t += (long long)gridDim.x * blockDim.x) {
        const long long n0 = base[t] / Q, n1 = n0 + nf[t];
        for (long long n = (n0 + 63) & ~63LL; n < n1; n += 64) unit_tile[n >> 6] = (int)t;
    }
}

// {low 32 bits of the block offset, count} of neighbour entry k of tile t
__global__ void entries_kernel(const int *nbr, const long long *base, const int *nf,
                               long long t_n, uint2 *entries) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < t_n * NBR;
         i += (long long)gridDim.x * blockDim.x) {
        const long long t = i / NBR;
        const int nb = nbr[i];
        const long long tt = nb >= 0 ? nb : t;
        entries[i] = make_uint2((unsigned)base[tt], (unsigned)nf[tt]);
    }
}

// one thread per slot: the node word + slot, and the ranks of the 18 pulled
// values in their source tiles
__global__ void node_records_kernel(const uint32_t *meta, const int *nbr, long long t_n,
                                    const long long *base, const unsigned char *rank,
                                    const int *unit_tile, uint32_t *node_meta,
                                    uint4 *node_rec) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < t_n * 64;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = rank[i];
        if (r == 255) continue;
        const long long t = i >> 6;
        const int j = (int)(i & 63);
        const long long n = base[t] / Q + r;
        const uint32_t m = meta[i];
        node_meta[n] = (m & 0x1ffffffu) | ((uint32_t)j << 25);
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        const int x = j & 3, y = (j >> 2) & 3, z = j >> 4;
        for (int q = 1; q < Q; ++q) {
            if (!((m >> q) & 1u)) {           // bounce-back: reads its own slot
                w[(q - 1) / 5] |= (uint32_t)r << (6 * ((q - 1) % 5));
                continue;
            }
            const int sx = x - ex(q), sy = y - ey(q), sz = z - ez(q);
            const int dx = sx < 0 ? -1 : (sx > 3 ? 1 : 0);
            const int dy = sy < 0 ? -1 : (sy > 3 ? 1 : 0);
            const int dz = sz < 0 ? -1 : (sz > 3 ? 1 : 0);
            const int k = delta_index(dx, dy, dz);
            const int nb = k == 13 ? (int)t : nbr[t * NBR + k];
            const int src = (sx & 3) + 4 * (sy & 3) + 16 * (sz & 3);
            const uint32_t rs = rank[(long long)nb * 64 + src] & 63u;
            w[(q - 1) / 5] |= rs << (6 * ((q - 1) % 5));
        }
        w[3] |= (uint32_t)r << 18;
        w[3] |= (uint32_t)(t - unit_tile[n >> 6]) << 24;
        node_rec[n] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

}  // namespace
}  // namespace tlbm

extern "C" int tlbm_compact_nodes(const uint32_t *d_meta, const int32_t *d_nbr, int64_t t_n,
                                  int64_t n_fn, const int64_t *d_base, const int32_t *d_nf,
                                  const uint8_t *d_rank, uint32_t *d_node_meta,
                                  uint32_t *d_node_rec, int32_t *d_unit_tile,
                                  uint32_t *d_entries, void *stream) {
    if (t_n == 0 || n_fn == 0) return TLBM_OK;
    if (!d_meta || !d_nbr || !d_base || !d_nf || !d_rank || !d_node_meta || !d_node_rec ||
        !d_unit_tile || !d_entries || t_n < 0 || n_fn < 0) {
        set_error("tlbm_compact_nodes: bad argument");
        return TLBM_ERR_ARG;
    }
    if ((long long)Q * n_fn >= (1LL << 32)) {
        set_error("tlbm_compact_nodes: 19 * n_fn = %lld needs 64-bit offsets",
                  (long long)Q * n_fn);
        return TLBM_ERR_ARG;
    }
    cudaStream_t s = as_stream(stream);
    const auto *base = reinterpret_cast<const long long *>(d_base);
    unit_tile_kernel<<<grid_for_slots(t_n), 256, 0, s>>>(base, d_nf, t_n, d_unit_tile);
    int rc = launch_check("unit_tile_kernel");
    if (rc) return rc;
    entries_kernel<<<grid_for_slots(t_n * NBR), 256, 0, s>>>(
        d_nbr, base, d_nf, t_n, reinterpret_cast<uint2 *>(d_entries));
    if ((rc = launch_check("entries_kernel"))) return rc;
    node_records_kernel<<<grid_for_slots(t_n * 64), 256, 0, s>>>(
        d_meta, d_nbr, t_n, base, d_rank, d_unit_tile, d_node_meta,
        reinterpret_cast<uint4 *>(d_node_rec));
    return launch_check("node_records_kernel");
}

// ---- slab halo on a compact store (fields.cu: halo_kernel for blocks) -----
// Same packed buffer as tlbm_halo -- buf[(tile - tile_begin) * 80 + k * 16 +
// (x + 4 y)] for the 5 directions crossing the outer z plane -- with each
// value found at base + q * nf + rank; solid slots pack as 0 and are skipped
// on unpack.
namespace tlbm {
namespace {

__host__ __device__ constexpr int compact_halo_dir(int up, int k) {
    return up ? (k == 0 ? 5 : k == 1 ? 11 : k == 2 ? 13 : k == 3 ? 15 : 17)
              : (k == 0 ? 6 : k == 1 ? 12 : k == 2 ? 14 : k == 3 ? 16 : 18);
}

template <class T, bool UP, bool PACK>
__global__ void halo_compact_kernel(T *f, long long tile_begin, long long n_tiles, T *buf,
                                    const long long *base, const int *nf,
                                    const unsigned char *rank) {
    const long long n = n_tiles * 80;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long t = tile_begin + i / 80;
        const int r = (int)(i % 80);
        const int k = r >> 4, s = r & 15;
        const int j = s + 16 * (UP ? 3 : 0);
        const int rk = rank[t * 64 + j];
        int q = 0;
#pragma unroll
        for (int kk = 0; kk < 5; ++kk)
            if (kk == k) q = compact_halo_dir(UP, kk);
        if (rk == 255) {
            if (PACK) buf[i] = T(0);
            continue;
        }
        const long long at = base[t] + (long long)q * nf[t] + rk;
        if (PACK) buf[i] = f[at];
        else f[at] = buf[i];
    }
}

template <class T>
int halo_compact_as(void *d_f, int64_t tile_begin, int64_t nt, int up, int pack, void *d_buf,
                    const int64_t *d_base, const int32_t *d_nf, const uint8_t *d_rank,
                    cudaStream_t s) {
    auto *f = static_cast<T *>(d_f);
    auto *b = static_cast<T *>(d_buf);
    const auto *base = reinterpret_cast<const long long *>(d_base);
    const unsigned g = grid_for_slots(nt * 80);
    if (up && pack) halo_compact_kernel<T, true, true><<<g, 256, 0, s>>>(f, tile_begin, nt, b, base, d_nf, d_rank);
    else if (up) halo_compact_kernel<T, true, false><<<g, 256, 0, s>>>(f, tile_begin, nt, b, base, d_nf, d_rank);
    else if (pack) halo_compact_kernel<T, false, true><<<g, 256, 0, s>>>(f, tile_begin, nt, b, base, d_nf, d_rank);
    else halo_compact_kernel<T, false, false><<<g, 256, 0, s>>>(f, tile_begin, nt, b, base, d_nf, d_rank);
    return launch_check("halo_compact_kernel");
}

}  // namespace
}  // namespace tlbm

extern "C" int tlbm_halo_compact(void *d_f, int dtype, int64_t tile_begin, int64_t tile_end,
                                 int up, int pack, void *d_buf, const int64_t *d_base,
                                 const int32_t *d_nf, const uint8_t *d_rank, void *stream) {
    if (tile_end < tile_begin || tile_begin < 0) {
        set_error("tlbm_halo_compact: bad tile range");
        return TLBM_ERR_ARG;
    }
    const long long nt = tile_end - tile_begin;
    if (nt == 0) return TLBM_OK;
    int rc;
    if ((rc = check_dtype(dtype))) return rc;
    if (!d_f || !d_buf || !d_base || !d_nf || !d_rank) {
        set_error("tlbm_halo_compact: null argument");
        return TLBM_ERR_ARG;
    }
    cudaStream_t s = as_stream(stream);
    return dtype == TLBM_F64
               ? halo_compact_as<double>(d_f, tile_begin, nt, up, pack, d_buf, d_base, d_nf, d_rank, s)
               : halo_compact_as<float>(d_f, tile_begin, nt, up, pack, d_buf, d_base, d_nf, d_rank, s);
}
