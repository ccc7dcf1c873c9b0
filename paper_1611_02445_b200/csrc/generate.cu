// GPU side of the sphere-pack generator (geometry.py:200-269 semantics,
// SURVEY §8f-3): for a batch of sphere centres, every voxel records the
// index of the first sphere that covers it (atomicMin).  The host turns the
// per-index counts into the solid fraction after k spheres and finds the
// reference's stopping sphere and pass acceptance exactly; the voxel test is
// the reference's float64 expression ((x+0.5-c0)^2 + (y+0.5-c1)^2) +
// (z+0.5-c2)^2 <= r^2 (library built with -fmad=false), so the result is
// bit-identical to geometry.generate_sphere_pack on the CPU.  The vessel
// tree generator (geometry.generate_vessel_tree(device=...)) rasterises the
// host-computed branch discs and classifies wall / fluid / inlet / outlet
// the same way, also bit-identically.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "d3q19.cuh"

namespace tlbm {
namespace {

__global__ void sphere_cover_kernel(const double *centres, long long first_index, int n,
                                    double rr, double r, int *first) {
    const long long s = blockIdx.x;
    const double c0 = centres[3 * s], c1 = centres[3 * s + 1], c2 = centres[3 * s + 2];
    // candidate box: every voxel whose centre can be within r of c, widened
    // by one voxel; the exact test below decides
    int lo[3], hi[3];
    const double c[3] = {c0, c1, c2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = max(0, (int)floor(c[k] - r - 0.5) - 1);
        hi[k] = min(n - 1, (int)ceil(c[k] + r - 0.5) + 1);
    }
    const int ex = hi[0] - lo[0] + 1, ey = hi[1] - lo[1] + 1, ez = hi[2] - lo[2] + 1;
    if (ex <= 0 || ey <= 0 || ez <= 0) return;
    const long long vol = (long long)ex * ey * ez;
    const int idx = (int)(first_index + s);
    for (long long v = threadIdx.x; v < vol; v += blockDim.x) {
        const int z = lo[2] + (int)(v % ez);
        const int y = lo[1] + (int)((v / ez) % ey);
        const int x = lo[0] + (int)(v / ((long long)ez * ey));
        const double dx = (x + 0.5) - c0, dy = (y + 0.5) - c1, dz = (z + 0.5) - c2;
        if ((dx * dx + dy * dy) + dz * dz <= rr)
            atomicMin(first + ((long long)x * n + y) * n + z, idx);
    }
}

// Vessel tree (geometry.generate_vessel_tree): lumen bytes per voxel from
// the per-z disc list the host computes (cx, cy, r per branch; the reference
// expression dx*dx + dy*dy <= r*r in float64), x/y margins cleared.
__global__ void vessel_lumen_kernel(const double *discs, const int32_t *count, int nb, int nx,
                                    int ny, int nz, int margin, uint8_t *lumen) {
    const long long total = (long long)nx * ny * nz;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x) {
        const int z = (int)(v % nz);
        const int y = (int)((v / nz) % ny);
        const int x = (int)(v / ((long long)nz * ny));
        uint8_t in = 0;
        if (x >= margin && x < nx - margin && y >= margin && y < ny - margin) {
            const double *d = discs + (long long)z * nb * 3;
            for (int i = 0; i < count[z]; ++i) {
                const double dx = (double)x - d[3 * i], dy = (double)y - d[3 * i + 1];
                const double r = d[3 * i + 2];
                if (dx * dx + dy * dy <= r * r) in = 1;
            }
        }
        lumen[v] = in;
    }
}

// Lumen voxels with all six neighbours in the lumen are FLUID, the rest
// BB_WALL; outside the box x/y count as solid and z replicates the end
// planes (open faces).  FLUID on z = 0 becomes INLET, on z = nz-1 OUTLET.
__global__ void vessel_types_kernel(const uint8_t *lumen, int nx, int ny, int nz, uint8_t *t) {
    const long long total = (long long)nx * ny * nz;
    const long long sx = (long long)ny * nz;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
         v += (long long)gridDim.x * blockDim.x) {
        const int z = (int)(v % nz);
        const int y = (int)((v / nz) % ny);
        const int x = (int)(v / sx);
        uint8_t tag = SOLID;
        if (lumen[v]) {
            const bool interior = x > 0 && lumen[v - sx] && x < nx - 1 && lumen[v + sx] &&
                                  y > 0 && lumen[v - nz] && y < ny - 1 && lumen[v + nz] &&
                                  (z == 0 || lumen[v - 1]) && (z == nz - 1 || lumen[v + 1]);
            tag = interior ? (z == 0 ? INLET : z == nz - 1 ? OUTLET : FLUID) : BB_WALL;
        }
        t[v] = tag;
    }
}

}  // namespace
}  // namespace tlbm

using namespace tlbm;

extern "C" int tlbm_sphere_cover(const double *d_centres, int64_t first_index, int64_t m, int n,
                                 double radius, int32_t *d_first, void *stream) {
    if (m < 0 || n < 1 || !(radius >= 0.0) || (m > 0 && (!d_centres || !d_first))) {
        set_error("tlbm_sphere_cover: bad argument");
        return TLBM_ERR_ARG;
    }
    if (m == 0) return TLBM_OK;
    sphere_cover_kernel<<<(unsigned)m, 256, 0, as_stream(stream)>>>(
        d_centres, (long long)first_index, n, radius * radius, radius, d_first);
    return launch_check("sphere_cover_kernel");
}

extern "C" int tlbm_vessel_tree(const double *d_discs, const int32_t *d_count, int nb, int nx,
                                int ny, int nz, int margin, uint8_t *d_lumen, uint8_t *d_types,
                                void *stream) {
    if (nb < 1 || nx < 1 || ny < 1 || nz < 1 || margin < 0 || !d_discs || !d_count ||
        !d_lumen || !d_types) {
        set_error("tlbm_vessel_tree: bad argument");
        return TLBM_ERR_ARG;
    }
    const long long total = (long long)nx * ny * nz;
    const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 64);
    cudaStream_t s = as_stream(stream);
    vessel_lumen_kernel<<<grid, 256, 0, s>>>(d_discs, d_count, nb, nx, ny, nz, margin, d_lumen);
    int rc = launch_check("vessel_lumen_kernel");
    if (rc != TLBM_OK) return rc;
    vessel_types_kernel<<<grid, 256, 0, s>>>(d_lumen, nx, ny, nz, d_types);
    return launch_check("vessel_types_kernel");
}
