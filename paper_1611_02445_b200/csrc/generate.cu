// GPU side of the sphere-pack generator (geometry.py:200-269 semantics,
// SURVEY §8f-3): for a batch of sphere centres, every voxel records the
// index of the first sphere that covers it (atomicMin).  The host turns the
// per-index counts into the solid fraction after k spheres and finds the
// reference's stopping sphere and pass acceptance exactly; the voxel test is
// the reference's float64 expression ((x+0.5-c0)^2 + (y+0.5-c1)^2) +
// (z+0.5-c2)^2 <= r^2 (library built with -fmad=false), so the result is
// bit-identical to geometry.generate_sphere_pack on the CPU.
#include <cmath>

#include "common.cuh"

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
