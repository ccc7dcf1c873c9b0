// Device tiler: Alg. 1 of the paper as the reference
// restates it in tiling.py:51-83, plus the neighbour-tile map
// (txmodel.py:145-160) and the per-slot node metadata the step kernel reads.
//
// tile_map construction is three kernels:
//   1. mark      -- coalesced pass over the uint8 voxel grid (one thread per
//                   4-voxel z-run); a run with any non-solid voxel marks its
//                   tile occupied (benign same-value stores).
//   2. reduce    -- occupied-tile count per 4096-tile chunk of the scan order
//                   (z outer, y, x inner).
//   3. scan      -- one CTA turns the chunk counts into exclusive offsets.
//   4. compact   -- each chunk rescans its flags and writes tile indices, so
//                   the numbering is order-stable exactly like
//                   np.flatnonzero(occupied.transpose(2, 1, 0).ravel()).
#include "common.cuh"
#include "d3q19.cuh"

namespace tlbm {
namespace {

constexpr int CHUNK_THREADS = 256;
constexpr int PER_THREAD = 16;
constexpr int CHUNK = CHUNK_THREADS * PER_THREAD;

struct Mesh {
    int nx, ny, nz, ntx, nty, ntz;
    __host__ __device__ long long tiles() const { return (long long)ntx * nty * ntz; }
};

__global__ void mark_kernel(const uint8_t *__restrict__ types, Mesh m,
                            uint8_t *__restrict__ occ) {
    long long runs = (long long)m.nx * m.ny * m.ntz;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < runs;
         r += (long long)gridDim.x * blockDim.x) {
        int tz = (int)(r % m.ntz);
        long long xy = r / m.ntz;
        int y = (int)(xy % m.ny);
        int x = (int)(xy / m.ny);
        const uint8_t *row = types + xy * m.nz;
        int z0 = 4 * tz;
        bool any = false;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (z0 + k < m.nz) any |= row[z0 + k] != 0;
        if (any) {
            long long l = (x >> 2) + (long long)m.ntx * ((y >> 2) + (long long)m.nty * tz);
            occ[l] = 1;
        }
    }
}

__device__ __forceinline__ int block_exclusive_scan(int v, int *smem, int *total) {
    // Kogge-Stone over the CTA via warp shuffles + one smem pass
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int nw = blockDim.x >> 5;
        int s = lane < nw ? smem[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) smem[lane] = s;
    }
    __syncthreads();
    int before = (warp > 0 ? smem[warp - 1] : 0) + x - v;
    if (total) *total = smem[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

__global__ void reduce_kernel(const uint8_t *__restrict__ occ, long long n,
                              int *__restrict__ chunk_sums) {
    __shared__ int smem[32];
    long long base = (long long)blockIdx.x * CHUNK + (long long)threadIdx.x * PER_THREAD;
    int c = 0;
#pragma unroll
    for (int i = 0; i < PER_THREAD; ++i)
        if (base + i < n) c += occ[base + i];
    int total;
    block_exclusive_scan(c, smem, &total);
    if (threadIdx.x == 0) chunk_sums[blockIdx.x] = total;
}

__global__ void scan_chunks_kernel(int *__restrict__ sums, int nchunks,
                                   long long *__restrict__ total) {
    __shared__ int smem[32];
    long long carry = 0;
    for (int base = 0; base < nchunks; base += blockDim.x) {
        int i = base + threadIdx.x;
        int v = i < nchunks ? sums[i] : 0;
        int tot;
        int ex = block_exclusive_scan(v, smem, &tot);
        if (i < nchunks) sums[i] = (int)(carry + ex);
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void compact_kernel(const uint8_t *__restrict__ occ, Mesh m,
                               const int *__restrict__ chunk_offsets,
                               int32_t *__restrict__ tile_map) {
    __shared__ int smem[32];
    long long n = m.tiles();
    long long base = (long long)blockIdx.x * CHUNK + (long long)threadIdx.x * PER_THREAD;
    uint8_t f[PER_THREAD];
    int c = 0;
#pragma unroll
    for (int i = 0; i < PER_THREAD; ++i) {
        f[i] = (base + i < n) ? occ[base + i] : 0;
        c += f[i];
    }
    int idx = chunk_offsets[blockIdx.x] + block_exclusive_scan(c, smem, nullptr);
#pragma unroll
    for (int i = 0; i < PER_THREAD; ++i) {
        long long l = base + i;
        if (l >= n) break;
        int tx = (int)(l % m.ntx);
        long long r = l / m.ntx;
        int ty = (int)(r % m.nty);
        int tz = (int)(r / m.nty);
        long long cm = ((long long)tx * m.nty + ty) * m.ntz + tz;
        tile_map[cm] = f[i] ? idx : -1;
        idx += f[i];
    }
}

__global__ void list_kernel(const int32_t *__restrict__ tile_map, Mesh m,
                            int32_t *__restrict__ non_empty) {
    long long n = m.tiles();
    for (long long cm = blockIdx.x * (long long)blockDim.x + threadIdx.x; cm < n;
         cm += (long long)gridDim.x * blockDim.x) {
        int v = tile_map[cm];
        if (v < 0) continue;
        int tz = (int)(cm % m.ntz);
        long long r = cm / m.ntz;
        int ty = (int)(r % m.nty);
        int tx = (int)(r / m.nty);
        non_empty[3LL * v + 0] = 4 * tx;
        non_empty[3LL * v + 1] = 4 * ty;
        non_empty[3LL * v + 2] = 4 * tz;
    }
}

__global__ void neighbor_kernel(const int32_t *__restrict__ tile_map, Mesh m,
                                const int32_t *__restrict__ non_empty, long long t_n,
                                int periodic, int32_t *__restrict__ nbr) {
    long long n = t_n * NBR;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        long long t = i / NBR;
        int k = (int)(i % NBR);
        int d[3] = {k / 9 - 1, (k / 3) % 3 - 1, k % 3 - 1};
        int dims[3] = {m.ntx, m.nty, m.ntz};
        int c[3];
        bool ok = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            c[a] = non_empty[3 * t + a] / 4 + d[a];
            if (periodic >> a & 1) c[a] = (c[a] + dims[a]) % dims[a];
            ok &= c[a] >= 0 && c[a] < dims[a];
        }
        nbr[i] = ok ? tile_map[((long long)c[0] * m.nty + c[1]) * m.ntz + c[2]] : -1;
    }
}

__global__ void meta_kernel(const uint8_t *__restrict__ types, Mesh m, int periodic,
                            const int32_t *__restrict__ non_empty, long long t_n,
                            uint32_t *__restrict__ meta, int32_t *__restrict__ bad) {
    long long n = t_n * 64;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        long long t = i >> 6;
        int j = (int)(i & 63);
        int p[3] = {non_empty[3 * t] + (j & 3), non_empty[3 * t + 1] + ((j >> 2) & 3),
                    non_empty[3 * t + 2] + (j >> 4)};
        int dims[3] = {m.nx, m.ny, m.nz};
        uint32_t w = 0;
        if (p[0] < m.nx && p[1] < m.ny && p[2] < m.nz) {
            int tag = types[((long long)p[0] * m.ny + p[1]) * m.nz + p[2]];
            if (tag > OUTLET) atomicAdd(bad + 1, 1);
            if (tag != SOLID) {
                w = META_ACTIVE | ((uint32_t)tag << 19);
#pragma unroll
                for (int q = 1; q < Q; ++q) {
                    int s[3] = {p[0] - ex(q), p[1] - ey(q), p[2] - ez(q)};
                    bool ok = true;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        if (periodic >> a & 1) s[a] = (s[a] + dims[a]) % dims[a];
                        ok &= s[a] >= 0 && s[a] < dims[a];
                    }
                    if (ok && types[((long long)s[0] * m.ny + s[1]) * m.nz + s[2]] != SOLID)
                        w |= 1u << q;
                }
                if (tag == INLET || tag == OUTLET) {
                    int cnt = 0, face = 0;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        if (periodic >> a & 1) continue;
                        if (p[a] == 0) { ++cnt; face = 2 * a; }
                        if (p[a] == dims[a] - 1) { ++cnt; face = 2 * a + 1; }
                    }
                    if (cnt != 1) atomicAdd(bad, 1);
                    w |= (uint32_t)face << 22;
                }
            }
        }
        meta[i] = w;
    }
}

__global__ void count_kernel(const uint32_t *__restrict__ meta, long long t_n,
                             int32_t *__restrict__ counts) {
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= t_n) return;
    uint32_t a = meta[warp * 64 + lane] & META_ACTIVE;
    uint32_t b = meta[warp * 64 + 32 + lane] & META_ACTIVE;
    int c = __popc(__ballot_sync(0xffffffffu, a)) + __popc(__ballot_sync(0xffffffffu, b));
    if (lane == 0) counts[warp] = c;
}

unsigned capped_grid(long long n, int block) {
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 148LL * 64) g = 148LL * 64;
    return (unsigned)g;
}

Mesh make_mesh(int nx, int ny, int nz) {
    return Mesh{nx, ny, nz, (nx + 3) / 4, (ny + 3) / 4, (nz + 3) / 4};
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace
}  // namespace tlbm

using namespace tlbm;

extern "C" size_t tlbm_tiling_scratch_bytes(int nx, int ny, int nz) {
    Mesh m = make_mesh(nx, ny, nz);
    long long n = m.tiles();
    long long nchunks = (n + CHUNK - 1) / CHUNK;
    return align256((size_t)n) + align256(sizeof(int) * (size_t)(nchunks + 1)) + 256;
}

extern "C" int tlbm_tile_map(const uint8_t *d_types, int nx, int ny, int nz,
                             int32_t *d_tile_map, void *d_scratch, int64_t *h_t_n,
                             void *stream) {
    if (nx < 1 || ny < 1 || nz < 1 || !d_types || !d_tile_map || !d_scratch || !h_t_n) {
        set_error("tlbm_tile_map: bad arguments");
        return TLBM_ERR_ARG;
    }
    cudaStream_t s = as_stream(stream);
    Mesh m = make_mesh(nx, ny, nz);
    long long n = m.tiles();
    long long nchunks = (n + CHUNK - 1) / CHUNK;
    uint8_t *occ = static_cast<uint8_t *>(d_scratch);
    int *sums = reinterpret_cast<int *>(occ + align256((size_t)n));
    long long *total = reinterpret_cast<long long *>(
        reinterpret_cast<char *>(sums) + align256(sizeof(int) * (size_t)(nchunks + 1)));
    int rc;
    if ((rc = cuda_check(cudaMemsetAsync(occ, 0, (size_t)n, s), "memset occupancy"))) return rc;
    mark_kernel<<<capped_grid((long long)nx * ny * m.ntz, 256), 256, 0, s>>>(d_types, m, occ);
    if ((rc = launch_check("mark_kernel"))) return rc;
    reduce_kernel<<<(unsigned)nchunks, CHUNK_THREADS, 0, s>>>(occ, n, sums);
    if ((rc = launch_check("reduce_kernel"))) return rc;
    scan_chunks_kernel<<<1, 1024, 0, s>>>(sums, (int)nchunks, total);
    if ((rc = launch_check("scan_chunks_kernel"))) return rc;
    compact_kernel<<<(unsigned)nchunks, CHUNK_THREADS, 0, s>>>(occ, m, sums, d_tile_map);
    if ((rc = launch_check("compact_kernel"))) return rc;
    long long t_n = 0;
    if ((rc = cuda_check(cudaMemcpyAsync(&t_n, total, sizeof(t_n), cudaMemcpyDeviceToHost, s),
                         "copy t_n")))
        return rc;
    if ((rc = cuda_check(cudaStreamSynchronize(s), "tile_map sync"))) return rc;
    *h_t_n = t_n;
    return TLBM_OK;
}

extern "C" int tlbm_tile_list(const int32_t *d_tile_map, int ntx, int nty, int ntz,
                              int32_t *d_non_empty, int64_t t_n, void *stream) {
    if (t_n == 0) return TLBM_OK;
    Mesh m{4 * ntx, 4 * nty, 4 * ntz, ntx, nty, ntz};
    list_kernel<<<capped_grid(m.tiles(), 256), 256, 0, as_stream(stream)>>>(d_tile_map, m,
                                                                          d_non_empty);
    return launch_check("list_kernel");
}

extern "C" int tlbm_tile_neighbors(const int32_t *d_tile_map, int ntx, int nty, int ntz,
                                   const int32_t *d_non_empty, int64_t t_n, int periodic_mask,
                                   int32_t *d_nbr, void *stream) {
    if (t_n == 0) return TLBM_OK;
    Mesh m{4 * ntx, 4 * nty, 4 * ntz, ntx, nty, ntz};
    neighbor_kernel<<<capped_grid(t_n * NBR, 256), 256, 0, as_stream(stream)>>>(
        d_tile_map, m, d_non_empty, t_n, periodic_mask, d_nbr);
    return launch_check("neighbor_kernel");
}

extern "C" int tlbm_node_meta(const uint8_t *d_types, int nx, int ny, int nz, int periodic_mask,
                              const int32_t *d_non_empty, int64_t t_n, uint32_t *d_meta,
                              int32_t *d_bad, void *stream) {
    if (t_n == 0) return TLBM_OK;
    Mesh m = make_mesh(nx, ny, nz);
    meta_kernel<<<capped_grid(t_n * 64, 256), 256, 0, as_stream(stream)>>>(
        d_types, m, periodic_mask, d_non_empty, t_n, d_meta, d_bad);
    return launch_check("meta_kernel");
}

extern "C" int tlbm_tile_counts(const uint32_t *d_meta, int64_t t_n, int32_t *d_counts,
                                void *stream) {
    if (t_n == 0) return TLBM_OK;
    count_kernel<<<grid_for(t_n * 32, 256), 256, 0, as_stream(stream)>>>(d_meta, t_n, d_counts);
    return launch_check("count_kernel");
}
