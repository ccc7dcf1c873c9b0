// Field-store kernels: equilibrium initialisation, canonical
// scatter/gather (layout.py:155-167) and the macroscopic readout
// (collision.py:75-121) -- all in the reference's arithmetic order.
#include <cmath>

#include "common.cuh"
#include "physics.cuh"

namespace tlbm {
namespace {

constexpr int TILE_VALUES = Q * 64;

__device__ __forceinline__ long long gtid() {
    return blockIdx.x * (long long)blockDim.x + threadIdx.x;
}
__device__ __forceinline__ long long gstride() { return (long long)gridDim.x * blockDim.x; }

unsigned grid_capped(long long n) {
    long long g = (n + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148LL * 32) g = 148LL * 32;
    return (unsigned)g;
}

template <class T, int QUASI, int TABLE>
__global__ void init_uniform_kernel(T *f, long long t_n, double rho_d, double ux, double uy,
                                    double uz) {
    for (long long i = gtid(); i < t_n * 64; i += gstride()) {
        const long long t = i >> 6;
        const int j = (int)(i & 63);
        const T rho = T(rho_d);
        const T u[3] = {T(ux), T(uy), T(uz)};
        const T usq = speed_sq(u);
#pragma unroll
        for (int q = 0; q < Q; ++q)
            f[t * TILE_VALUES + q * 64 + slot_of<TABLE>(q, j & 3, (j >> 2) & 3, j >> 4)] =
                equilibrium_q<T, QUASI>(q, rho, u, usq);
    }
}

template <class T, int QUASI, int TABLE>
__global__ void init_fields_kernel(T *f, long long t_n, const T *rho, const T *u) {
    const long long n = t_n * 64;
    for (long long i = gtid(); i < n; i += gstride()) {
        const long long t = i >> 6;
        const int j = (int)(i & 63);
        const T r = rho[i];
        const T uu[3] = {u[i], u[n + i], u[2 * n + i]};
        const T usq = speed_sq(uu);
#pragma unroll
        for (int q = 0; q < Q; ++q)
            f[t * TILE_VALUES + q * 64 + slot_of<TABLE>(q, j & 3, (j >> 2) & 3, j >> 4)] =
                equilibrium_q<T, QUASI>(q, r, uu, usq);
    }
}

template <class T, int TABLE, bool TO_CANON>
__global__ void canon_kernel(const T *in, T *out, long long t_n) {
    const long long n = t_n * 64;
    for (long long i = gtid(); i < n; i += gstride()) {
        const long long t = i >> 6;
        const int j = (int)(i & 63);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const long long blk = t * TILE_VALUES + q * 64 + slot_of<TABLE>(q, j & 3, (j >> 2) & 3, j >> 4);
            const long long can = q * n + i;
            if (TO_CANON) out[can] = in[blk];
            else out[blk] = in[can];
        }
    }
}

template <class T, int QUASI>
__device__ __forceinline__ uint32_t readout(const T (&g)[Q], long long i, long long n, T *rho,
                                            T *u, T *p) {
    T r, uu[3];
    moments<T, QUASI>(g, r, uu);
    rho[i] = r;
    u[i] = uu[0];
    u[n + i] = uu[1];
    u[2 * n + i] = uu[2];
    if (p) p[i] = r / T(3.0);
    return status_of<T, QUASI>(r, T(0), T(HUGE_VAL));
}

template <class T, int QUASI, int TABLE>
__global__ void macro_blocks_kernel(const T *f, long long t_n, T *rho, T *u, T *p,
                                    uint32_t *flags) {
    const long long n = t_n * 64;
    uint32_t st = 0;
    for (long long i = gtid(); i < n; i += gstride()) {
        const long long t = i >> 6;
        const int j = (int)(i & 63);
        T g[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q)
            g[q] = f[t * TILE_VALUES + q * 64 + slot_of<TABLE>(q, j & 3, (j >> 2) & 3, j >> 4)];
        st |= readout<T, QUASI>(g, i, n, rho, u, p);
    }
    if (flags && st) atomicOr(flags, st);
}

template <class T, int QUASI>
__global__ void macro_canon_kernel(const T *f, long long n, T *rho, T *u, T *p,
                                   uint32_t *flags) {
    uint32_t st = 0;
    for (long long i = gtid(); i < n; i += gstride()) {
        T g[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) g[q] = f[q * n + i];
        st |= readout<T, QUASI>(g, i, n, rho, u, p);
    }
    if (flags && st) atomicOr(flags, st);
}

template <class T, int QUASI>
__global__ void equilibrium_kernel(const T *rho, const T *u, long long n, T *feq) {
    for (long long i = gtid(); i < n; i += gstride()) {
        const T uu[3] = {u[i], u[n + i], u[2 * n + i]};
        const T usq = speed_sq(uu);
#pragma unroll
        for (int q = 0; q < Q; ++q) feq[q * n + i] = equilibrium_q<T, QUASI>(q, rho[i], uu, usq);
    }
}

template <class T>
struct OpParam {
    T op[Q * Q];
};

template <class T, int QUASI>
__global__ void collide_mrt_kernel(T *f, long long n, const OpParam<T> op, uint32_t *flags) {
    uint32_t st = 0;
    for (long long i = gtid(); i < n; i += gstride()) {
        T g[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) g[q] = f[q * n + i];
        st |= collide_mrt<T, QUASI>(g, op.op, T(HUGE_VAL));
#pragma unroll
        for (int q = 0; q < Q; ++q) f[q * n + i] = g[q];
    }
    if (flags && st) atomicOr(flags, st);
}

// apply_operator (collision.py:216-231): out[i] = sum over j with op[i][j]
// != 0, in j order, of op[i][j] * delta[j].  WIDE (float32 data, float64
// operator): NumPy evaluates `acc += c * delta[j]` with a float64 scalar c
// in float64 and rounds into the float32 accumulator (NEP 50), so each term
// and partial sum is formed in double and rounded to T after every add.
template <class T, int WIDE>
__device__ __forceinline__ void apply_op_column(const double *op, const T (&d)[Q], T (&out)[Q]) {
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        T acc = T(0);
        for (int j = 0; j < Q; ++j) {
            const double c = op[i * Q + j];
            if (c == 0.0) continue;
            if (WIDE) acc = T(double(acc) + c * double(d[j]));
            else acc = acc + T(c) * d[j];
        }
        out[i] = acc;
    }
}

template <class T, int WIDE>
__global__ void apply_operator_kernel(const T *delta, T *out, long long n,
                                      const OpParam<double> op) {
    for (long long i = gtid(); i < n; i += gstride()) {
        T d[Q], r[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) d[q] = delta[q * n + i];
        apply_op_column<T, WIDE>(op.op, d, r);
#pragma unroll
        for (int q = 0; q < Q; ++q) out[q * n + i] = r[q];
    }
}

// collide_mrt (collision.py:234-247) with a float64 operator on float32
// populations: f + apply_operator(op, feq - f) with the wide accumulation
template <int QUASI>
__global__ void collide_mrt_wide_kernel(float *f, long long n, const OpParam<double> op,
                                        uint32_t *flags) {
    uint32_t st = 0;
    for (long long i = gtid(); i < n; i += gstride()) {
        float g[Q], d[Q], r[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) g[q] = f[q * n + i];
        st |= mrt_deviations<float, QUASI>(g, d, float(HUGE_VAL));
        apply_op_column<float, 1>(op.op, d, r);
#pragma unroll
        for (int q = 0; q < Q; ++q) f[q * n + i] = g[q] + r[q];
    }
    if (flags && st) atomicOr(flags, st);
}

template <class T, int QUASI>
__global__ void collide_kernel(T *f, long long n, double inv_tau, uint32_t *flags) {
    uint32_t st = 0;
    for (long long i = gtid(); i < n; i += gstride()) {
        T g[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) g[q] = f[q * n + i];
        st |= collide<T, QUASI>(g, T(inv_tau), T(HUGE_VAL));
#pragma unroll
        for (int q = 0; q < Q; ++q) f[q * n + i] = g[q];
    }
    if (flags && st) atomicOr(flags, st);
}

template <class T, int QUASI, int FACE>
__device__ __forceinline__ T zou_he_node(T (&g)[Q], int kind, const double (&u_in)[3],
                                         double rho0) {
    // value returned by zou_he_velocity (implied rho) / zou_he_pressure (jn);
    // k0 and km are untouched by the closure (c.n <= 0)
    const T k0 = ordered_sum<T, FACE>(g, 0, -1, 0);
    const T km = ordered_sum<T, FACE>(g, -1, -1, 0);
    T ret;
    if (kind == 0) {
        const T un = T(face_sign(FACE)) * T(u_in[face_axis(FACE)]);
        ret = QUASI ? (k0 + T(2.0) * km) / (T(1.0) - un) : k0 + T(2.0) * km + un;
        zh_velocity<T, QUASI, FACE>(g, u_in);
    } else {
        ret = T(rho0) - (k0 + T(2.0) * km);
        zh_pressure<T, FACE>(g, rho0);
    }
    return ret;
}

template <class T, int QUASI, int FACE>
__global__ void zou_he_kernel(T *g_all, long long m, int kind, double ux, double uy, double uz,
                              double rho0, T *ret) {
    const double u_in[3] = {ux, uy, uz};
    for (long long i = gtid(); i < m; i += gstride()) {
        T g[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) g[q] = g_all[q * m + i];
        const T r = zou_he_node<T, QUASI, FACE>(g, kind, u_in, rho0);
#pragma unroll
        for (int q = 0; q < Q; ++q) g_all[q * m + i] = g[q];
        if (ret) ret[i] = r;
    }
}

}  // namespace
}  // namespace tlbm

using namespace tlbm;

extern "C" int tlbm_init_equilibrium(void *d_f, int dtype, int fluid, int table, int64_t t_n,
                                     double rho, double ux, double uy, double uz, void *stream) {
    if (t_n == 0) return TLBM_OK;
    return dispatch(dtype, fluid, table, [&]<class T, int QU, int TB>() {
        init_uniform_kernel<T, QU, TB><<<grid_capped(t_n * 64), 256, 0, as_stream(stream)>>>(
            static_cast<T *>(d_f), t_n, rho, ux, uy, uz);
        return launch_check("init_uniform_kernel");
    });
}

extern "C" int tlbm_init_from_macroscopic(void *d_f, int dtype, int fluid, int table, int64_t t_n,
                                          const void *d_rho, const void *d_u, void *stream) {
    if (t_n == 0) return TLBM_OK;
    return dispatch(dtype, fluid, table, [&]<class T, int QU, int TB>() {
        init_fields_kernel<T, QU, TB><<<grid_capped(t_n * 64), 256, 0, as_stream(stream)>>>(
            static_cast<T *>(d_f), t_n, static_cast<const T *>(d_rho),
            static_cast<const T *>(d_u));
        return launch_check("init_fields_kernel");
    });
}

extern "C" int tlbm_to_canonical(const void *d_f, int dtype, int table, int64_t t_n,
                                 void *d_canon, void *stream) {
    if (t_n == 0) return TLBM_OK;
    return dispatch(dtype, 0, table, [&]<class T, int QU, int TB>() {
        canon_kernel<T, TB, true><<<grid_capped(t_n * 64), 256, 0, as_stream(stream)>>>(
            static_cast<const T *>(d_f), static_cast<T *>(d_canon), t_n);
        return launch_check("canon_kernel");
    });
}

extern "C" int tlbm_from_canonical(const void *d_canon, int dtype, int table, int64_t t_n,
                                   void *d_f, void *stream) {
    if (t_n == 0) return TLBM_OK;
    return dispatch(dtype, 0, table, [&]<class T, int QU, int TB>() {
        canon_kernel<T, TB, false><<<grid_capped(t_n * 64), 256, 0, as_stream(stream)>>>(
            static_cast<const T *>(d_canon), static_cast<T *>(d_f), t_n);
        return launch_check("canon_kernel");
    });
}

extern "C" int tlbm_macroscopic(const void *d_f, int dtype, int fluid, int table, int64_t t_n,
                                void *d_rho, void *d_u, void *d_p, uint32_t *d_flags,
                                void *stream) {
    if (t_n == 0) return TLBM_OK;
    return dispatch(dtype, fluid, table, [&]<class T, int QU, int TB>() {
        macro_blocks_kernel<T, QU, TB><<<grid_capped(t_n * 64), 256, 0, as_stream(stream)>>>(
            static_cast<const T *>(d_f), t_n, static_cast<T *>(d_rho), static_cast<T *>(d_u),
            static_cast<T *>(d_p), d_flags);
        return launch_check("macro_blocks_kernel");
    });
}

extern "C" int tlbm_macroscopic_canonical(const void *d_f, int dtype, int fluid, int64_t n,
                                          void *d_rho, void *d_u, void *d_p, uint32_t *d_flags,
                                          void *stream) {
    if (n == 0) return TLBM_OK;
    return dispatch(dtype, fluid, 0, [&]<class T, int QU, int TB>() {
        macro_canon_kernel<T, QU><<<grid_capped(n), 256, 0, as_stream(stream)>>>(
            static_cast<const T *>(d_f), n, static_cast<T *>(d_rho), static_cast<T *>(d_u),
            static_cast<T *>(d_p), d_flags);
        return launch_check("macro_canon_kernel");
    });
}

extern "C" int tlbm_equilibrium(const void *d_rho, const void *d_u, int dtype, int fluid,
                                int64_t n, void *d_feq, void *stream) {
    if (n == 0) return TLBM_OK;
    return dispatch(dtype, fluid, 0, [&]<class T, int QU, int TB>() {
        equilibrium_kernel<T, QU><<<grid_capped(n), 256, 0, as_stream(stream)>>>(
            static_cast<const T *>(d_rho), static_cast<const T *>(d_u), n,
            static_cast<T *>(d_feq));
        return launch_check("equilibrium_kernel");
    });
}

extern "C" int tlbm_collide_lbgk(void *d_f, int dtype, int fluid, int64_t n, double tau,
                                 uint32_t *d_flags, void *stream) {
    if (n == 0) return TLBM_OK;
    return dispatch(dtype, fluid, 0, [&]<class T, int QU, int TB>() {
        collide_kernel<T, QU><<<grid_capped(n), 256, 0, as_stream(stream)>>>(
            static_cast<T *>(d_f), n, 1.0 / tau, d_flags);
        return launch_check("collide_kernel");
    });
}

extern "C" int tlbm_collide_mrt(void *d_f, int dtype, int fluid, int64_t n, const double *h_op,
                                uint32_t *d_flags, void *stream) {
    if (!h_op) {
        set_error("tlbm_collide_mrt: operator required");
        return TLBM_ERR_ARG;
    }
    if (n == 0) return TLBM_OK;
    return dispatch(dtype, fluid, 0, [&]<class T, int QU, int TB>() {
        OpParam<T> op;
        for (int k = 0; k < Q * Q; ++k) op.op[k] = T(h_op[k]);
        collide_mrt_kernel<T, QU><<<grid_capped(n), 256, 0, as_stream(stream)>>>(
            static_cast<T *>(d_f), n, op, d_flags);
        return launch_check("collide_mrt_kernel");
    });
}

extern "C" int tlbm_apply_operator(const void *d_delta, void *d_out, int dtype, int64_t n,
                                   const double *h_op, int wide, void *stream) {
    if (!h_op || !d_delta || !d_out) {
        set_error("tlbm_apply_operator: operator, input and output required");
        return TLBM_ERR_ARG;
    }
    if (n == 0) return TLBM_OK;
    OpParam<double> op;
    for (int k = 0; k < Q * Q; ++k) op.op[k] = h_op[k];
    return dispatch(dtype, 0, 0, [&]<class T, int QU, int TB>() {
        auto *in = static_cast<const T *>(d_delta);
        auto *out = static_cast<T *>(d_out);
        if (wide && sizeof(T) == 4)
            apply_operator_kernel<T, 1><<<grid_capped(n), 256, 0, as_stream(stream)>>>(
                in, out, n, op);
        else
            apply_operator_kernel<T, 0><<<grid_capped(n), 256, 0, as_stream(stream)>>>(
                in, out, n, op);
        return launch_check("apply_operator_kernel");
    });
}

extern "C" int tlbm_collide_mrt_wide(void *d_f, int fluid, int64_t n, const double *h_op,
                                     uint32_t *d_flags, void *stream) {
    if (!h_op) {
        set_error("tlbm_collide_mrt_wide: operator required");
        return TLBM_ERR_ARG;
    }
    if (n == 0) return TLBM_OK;
    OpParam<double> op;
    for (int k = 0; k < Q * Q; ++k) op.op[k] = h_op[k];
    return dispatch(TLBM_F32, fluid, 0, [&]<class T, int QU, int TB>() {
        collide_mrt_wide_kernel<QU><<<grid_capped(n), 256, 0, as_stream(stream)>>>(
            static_cast<float *>(d_f), n, op, d_flags);
        return launch_check("collide_mrt_wide_kernel");
    });
}

extern "C" int tlbm_zou_he(void *d_g, int dtype, int fluid, int face, int kind, int64_t m,
                           double ux, double uy, double uz, double rho0, void *d_ret,
                           void *stream) {
    if (face < 0 || face > 5 || (kind != 0 && kind != 1)) {
        set_error("tlbm_zou_he: face must be 0..5 and kind 0 (velocity) or 1 (pressure)");
        return TLBM_ERR_ARG;
    }
    if (m == 0) return TLBM_OK;
    return dispatch(dtype, fluid, 0, [&]<class T, int QU, int TB>() {
        auto *g = static_cast<T *>(d_g);
        auto *r = static_cast<T *>(d_ret);
        cudaStream_t s = as_stream(stream);
        unsigned gr = grid_capped(m);
        switch (face) {
            case 0: zou_he_kernel<T, QU, 0><<<gr, 256, 0, s>>>(g, m, kind, ux, uy, uz, rho0, r); break;
            case 1: zou_he_kernel<T, QU, 1><<<gr, 256, 0, s>>>(g, m, kind, ux, uy, uz, rho0, r); break;
            case 2: zou_he_kernel<T, QU, 2><<<gr, 256, 0, s>>>(g, m, kind, ux, uy, uz, rho0, r); break;
            case 3: zou_he_kernel<T, QU, 3><<<gr, 256, 0, s>>>(g, m, kind, ux, uy, uz, rho0, r); break;
            case 4: zou_he_kernel<T, QU, 4><<<gr, 256, 0, s>>>(g, m, kind, ux, uy, uz, rho0, r); break;
            default: zou_he_kernel<T, QU, 5><<<gr, 256, 0, s>>>(g, m, kind, ux, uy, uz, rho0, r); break;
        }
        return launch_check("zou_he_kernel");
    });
}

// ---- slab halo (multi-GPU z decomposition) --------------------
// A rank's boundary tile layer sends, per tile, the 16 nodes of its outer z
// plane for the 5 directions that cross it: up (e_z = +1: T, NT, ST, ET, WT)
// from plane z = 3, down (e_z = -1: B, NB, SB, EB, WB) from plane z = 0.
// Packed layout: buf[(tile - tile_begin) * 80 + k * 16 + (x + 4 y)].
namespace tlbm {
namespace {

__host__ __device__ constexpr int halo_dir(int up, int k) {
    return up ? (k == 0 ? 5 : k == 1 ? 11 : k == 2 ? 13 : k == 3 ? 15 : 17)
              : (k == 0 ? 6 : k == 1 ? 12 : k == 2 ? 14 : k == 3 ? 16 : 18);
}

template <class T, int TABLE, int UP, bool PACK>
__global__ void halo_kernel(T *f, long long tile_begin, long long n_tiles, T *buf) {
    const long long n = n_tiles * 80;
    for (long long i = gtid(); i < n; i += gstride()) {
        const long long t = i / 80;
        const int r = (int)(i % 80);
        const int k = r >> 4, s = r & 15;
        const int x = s & 3, y = s >> 2, z = UP ? 3 : 0;
        int q = 0;
#pragma unroll
        for (int kk = 0; kk < 5; ++kk)
            if (kk == k) q = halo_dir(UP, kk);
        int slot = 0;
#pragma unroll
        for (int kk = 0; kk < 5; ++kk)
            if (kk == k) slot = slot_of<TABLE>(halo_dir(UP, kk), x, y, z);
        const long long at = (tile_begin + t) * TILE_VALUES + q * 64 + slot;
        if (PACK) buf[i] = f[at];
        else f[at] = buf[i];
    }
}

}  // namespace
}  // namespace tlbm

extern "C" int tlbm_halo(void *d_f, int dtype, int table, int64_t tile_begin, int64_t tile_end,
                         int up, int pack, void *d_buf, void *stream) {
    if (tile_end < tile_begin || tile_begin < 0) {
        set_error("tlbm_halo: bad tile range");
        return TLBM_ERR_ARG;
    }
    const long long nt = tile_end - tile_begin;
    if (nt == 0) return TLBM_OK;
    return dispatch(dtype, 0, table, [&]<class T, int QU, int TB>() {
        auto *f = static_cast<T *>(d_f);
        auto *b = static_cast<T *>(d_buf);
        cudaStream_t s = as_stream(stream);
        unsigned g = grid_capped(nt * 80);
        if (up && pack) halo_kernel<T, TB, 1, true><<<g, 256, 0, s>>>(f, tile_begin, nt, b);
        else if (up) halo_kernel<T, TB, 1, false><<<g, 256, 0, s>>>(f, tile_begin, nt, b);
        else if (pack) halo_kernel<T, TB, 0, true><<<g, 256, 0, s>>>(f, tile_begin, nt, b);
        else halo_kernel<T, TB, 0, false><<<g, 256, 0, s>>>(f, tile_begin, nt, b);
        return launch_check("halo_kernel");
    });
}
