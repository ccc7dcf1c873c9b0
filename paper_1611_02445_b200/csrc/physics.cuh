// Node physics on register-resident populations g[19]: moments, LBGK
// collision and the Zou-He face closures.
//
// Every expression keeps the reference's operation order (collision.py:46-130,
// boundaries.py:132-195) and the library is compiled
// with -fmad=false, so no multiply-add is contracted: with IEEE division and
// square root (nvcc defaults) the results are bit-identical to the numpy
// reference and to the C oracle, in both fp64 and fp32.
//
// All direction indices are compile-time after loop unrolling, so g[] stays
// in registers (no local-memory indexing; checked with -Xptxas -v).
#pragma once
#include "d3q19.cuh"
#include "mrt_pattern.cuh"

#ifndef TLBM_MRT_GROUPED
#define TLBM_MRT_GROUPED 1
#endif

namespace tlbm {

enum : uint32_t { ST_DIVERGED = 1u, ST_GUARD = 2u };

// rho = ((g0 + g1) + ...) + g18; j_a accumulated from 0 in q order
// (collision.py:55-72); u = j / rho (quasi) or j (incompressible)
//
// The reference starts j and cu from 0 (np.zeros_like); "0 + x" is folded to
// x here.  That changes at most the sign of an exactly-zero partial sum,
// which never changes a post-collision population (every later use adds a
// non-negative term or squares it), so results stay bit-identical.
template <class T, int QUASI>
__device__ __forceinline__ void moments(const T (&g)[Q], T &rho, T (&u)[3]) {
    rho = g[0];
#pragma unroll
    for (int q = 1; q < Q; ++q) rho = rho + g[q];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        T acc = T(0);
        bool first = true;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int e = e_axis(q, a);
            if (e == 0) continue;
            if (first) acc = e > 0 ? g[q] : -g[q];
            else acc = e > 0 ? acc + g[q] : acc - g[q];
            first = false;
        }
        u[a] = QUASI ? acc / rho : acc;
    }
}

// collision.py:94-121 for one direction
template <class T, int QUASI>
__device__ __forceinline__ T equilibrium_q(int q, T rho, const T (&u)[3], T usq) {
    T cu = T(0);
    bool first = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int e = e_axis(q, a);
        if (e == 0) continue;
        const T term = e > 0 ? u[a] : -u[a];
        cu = first ? term : cu + term;
        first = false;
    }
    T br = T(3.0) * cu + T(4.5) * cu * cu - T(1.5) * usq;
    T w = T(weight(q));
    return QUASI ? w * (rho * (T(1.0) + br)) : w * (rho + br);
}

template <class T>
__device__ __forceinline__ T speed_sq(const T (&u)[3]) {
    return u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
}

// divergence: NaN, or rho <= 0 in the quasi-compressible model
// (collision.py:84-86); guard: |u|^2 > u_max_guard^2
template <class T, int QUASI>
__device__ __forceinline__ uint32_t status_of(T rho, T usq, T guard_sq) {
    uint32_t st = 0;
    if (rho != rho || (QUASI && !(rho > T(0)))) st |= ST_DIVERGED;
    if (usq > guard_sq) st |= ST_GUARD;
    return st;
}

// collide_lbgk in place: g <- g + fl(1/tau) (feq - g)  (collision.py:124-130)
//
// Opposite directions share their products: c.u of opp(q) is exactly -c.u of
// q, so 3 cu and (4.5 cu) cu are computed once per pair and the reference's
// bracket 3cu + 4.5cu*cu - 1.5usq becomes (A + B) - C for q and (B - A) - C
// for opp(q) -- the same IEEE results ((-A) + B == B - A), fewer instructions.
template <class T, int QUASI>
__device__ __forceinline__ T feq_of(int q, T rho, T br) {
    const T w = T(weight(q));
    return QUASI ? w * (rho * (T(1.0) + br)) : w * (rho + br);
}

// ---- fused multiply-add arithmetic (TLBM_ARITH_FMA) ------------------------
// The same LBGK / MRT maps with products contracted into FMAs:
//   bracket(q), bracket(opp q) = fma(+-3, cu, fma(4.5 cu, cu, -1.5 usq))
//   feq = fma(w, bracket, w rho)            (quasi: fma(w rho, bracket, w rho))
//   g  <- fma(1/tau, feq - g, g)
//   MRT: the operator applied in moment space (collide_mrt_fma below)
// 149 instead of 216 FP instructions per LBGK node and 218 instead of 722 for
// the MRT operator.  Every FMA rounds once where the reference rounds twice,
// so results differ from the reference in the last bits only; the parity bar
// is the stated 1e-12 tolerance (tests/test_gpu_fma.py: 2.7e-15 in f, 2.0e-14
// in u after 1000 cavity-64 steps).  fp64 only: in fp32 the same map drifts
// to 1.1e-5 in u, past the 1e-5 bar, so the step rejects it there.
template <class T>
__device__ __forceinline__ T fmad(T a, T b, T c) { return fma(a, b, c); }
template <>
__device__ __forceinline__ float fmad<float>(float a, float b, float c) { return fmaf(a, b, c); }

template <class T, int QUASI>
__device__ __forceinline__ T feq_fma(T wrho, T w, T br) {
    return QUASI ? fmad(wrho, br, wrho) : fmad(w, br, wrho);
}

// feq - g for all 19 directions into d[] (FMA arithmetic); returns status
template <class T, int QUASI>
__device__ __forceinline__ uint32_t deviations_fma(const T (&g)[Q], T (&d)[Q], T guard_sq) {
    T rho, u[3];
    moments<T, QUASI>(g, rho, u);
    const T usq = fmad(u[0], u[0], fmad(u[1], u[1], u[2] * u[2]));
    const T mc15 = T(-1.5) * usq;
    const T w0 = T(weight(0)), w1 = T(weight(1)), w7 = T(weight(7));
    const T wr0 = w0 * rho, wr1 = w1 * rho, wr7 = w7 * rho;
    d[0] = feq_fma<T, QUASI>(wr0, w0, mc15) - g[0];
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (opp(q) < q) continue;
        const int o = opp(q);
        T cu = T(0);
        bool first = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int e = e_axis(q, a);
            if (e == 0) continue;
            const T term = e > 0 ? u[a] : -u[a];
            cu = first ? term : cu + term;
            first = false;
        }
        const T P = fmad(T(4.5) * cu, cu, mc15);
        const T w = q <= 6 ? w1 : w7, wr = q <= 6 ? wr1 : wr7;
        d[q] = feq_fma<T, QUASI>(wr, w, fmad(T(3.0), cu, P)) - g[q];
        d[o] = feq_fma<T, QUASI>(wr, w, fmad(T(-3.0), cu, P)) - g[o];
    }
    return status_of<T, QUASI>(rho, usq, guard_sq);
}

template <class T, int QUASI>
__device__ __forceinline__ uint32_t collide_fma(T (&g)[Q], T inv_tau, T guard_sq) {
    T d[Q];
    const uint32_t st = deviations_fma<T, QUASI>(g, d, guard_sq);
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] = fmad(inv_tau, d[q], g[q]);
    return st;
}

// The D3Q19 moment basis of collision.py (MOMENT_MATRIX, collision.py:150-
// 160): integer coefficients of moment k on direction q.
__host__ __device__ constexpr int moment_coef(int k, int q) {
    const int x = ex(q), y = ey(q), z = ez(q);
    const int e2 = x * x + y * y + z * z;
    const int axx = 3 * x * x - e2, aww = y * y - z * z;
    switch (k) {
        case 0: return 1;
        case 1: return 19 * e2 - 30;
        case 2: return (21 * e2 * e2 - 53 * e2 + 24) / 2;
        case 3: return x;
        case 4: return (5 * e2 - 9) * x;
        case 5: return y;
        case 6: return (5 * e2 - 9) * y;
        case 7: return z;
        case 8: return (5 * e2 - 9) * z;
        case 9: return axx;
        case 10: return (3 * e2 - 5) * axx;
        case 11: return aww;
        case 12: return (3 * e2 - 5) * aww;
        case 13: return x * y;
        case 14: return y * z;
        case 15: return x * z;
        case 16: return aww * x;
        case 17: return (z * z - x * x) * y;
        default: return (x * x - y * y) * z;
    }
}
// moments of odd degree flip sign between q and opp(q)
__host__ __device__ constexpr bool moment_odd(int k) {
    return (k >= 3 && k <= 8) || k >= 16;
}
__host__ __device__ constexpr bool moment_conserved(int k) {
    return k == 0 || k == 3 || k == 5 || k == 7;
}
__host__ __device__ constexpr int moment_norm(int k) {
    int n = 0;
    for (int q = 0; q < Q; ++q) n += moment_coef(k, q) * moment_coef(k, q);
    return n;
}

// A coefficient-times-term with an integer coefficient: +-1 as add/sub, 0
// skipped, otherwise one FMA; the first term starts the sum.
template <class T>
__device__ __forceinline__ void acc_int(T &acc, bool &first, int c, T v) {
    if (c == 0) return;
    if (first) {
        acc = c == 1 ? v : c == -1 ? -v : T(c) * v;
        first = false;
    } else {
        acc = c == 1 ? acc + v : c == -1 ? acc - v : fmad(T(c), v, acc);
    }
}

// MRT in FMA arithmetic, in moment space: the operator is M^-1 diag(s) M in
// collision.py's basis with s = 0 on the conserved moments (the host checks
// that form, step_impl.cuh: mrt_moment_rates, and runs reference arithmetic
// for any other operator); w[k] = s_k / |M_k|^2.  Direction pairs split into
// sums (even moments) and differences (odd moments): 18 pair terms, 15
// projections with integer coefficients (83 add / FMA), 15 scalings, the
// transpose back (83) and 19 recombinations -- 218 DP instructions per node
// instead of the 380 of the dense FMA product.
template <class T, int QUASI>
__device__ __forceinline__ uint32_t collide_mrt_fma(T (&g)[Q], const T *w, T guard_sq) {
    T d[Q];
    const uint32_t st = deviations_fma<T, QUASI>(g, d, guard_sq);
    T sp[Q], dp[Q];
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (opp(q) < q) continue;
        sp[q] = d[q] + d[opp(q)];
        dp[q] = d[q] - d[opp(q)];
    }
    T y[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        if (moment_conserved(k)) continue;
        T m = T(0);
        bool first = true;
        if (!moment_odd(k)) acc_int(m, first, moment_coef(k, 0), d[0]);
#pragma unroll
        for (int q = 1; q < Q; ++q) {
            if (opp(q) < q) continue;
            acc_int(m, first, moment_coef(k, q), moment_odd(k) ? dp[q] : sp[q]);
        }
        y[k] = w[k] * m;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (q > 0 && opp(q) < q) continue;
        T ev = T(0), od = T(0);
        bool fe = true, fo = true;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            if (moment_conserved(k)) continue;
            if (moment_odd(k)) acc_int(od, fo, moment_coef(k, q), y[k]);
            else acc_int(ev, fe, moment_coef(k, q), y[k]);
        }
        if (q == 0) {
            g[0] = g[0] + ev;
        } else {
            g[q] = g[q] + (ev + od);
            g[opp(q)] = g[opp(q)] + (ev - od);
        }
    }
    return st;
}

template <class T, int QUASI>
__device__ __forceinline__ uint32_t collide(T (&g)[Q], T inv_tau, T guard_sq) {
    T rho, u[3];
    moments<T, QUASI>(g, rho, u);
    const T usq = speed_sq(u);
    const T c15 = T(1.5) * usq;
    {
        const T br = (T(3.0) * T(0) + T(4.5) * T(0) * T(0)) - c15;   // q = 0: cu = 0
        g[0] = g[0] + inv_tau * (feq_of<T, QUASI>(0, rho, br) - g[0]);
    }
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (opp(q) < q) continue;
        const int o = opp(q);
        T cu = T(0);
        bool first = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int e = e_axis(q, a);
            if (e == 0) continue;
            const T term = e > 0 ? u[a] : -u[a];
            cu = first ? term : cu + term;
            first = false;
        }
        const T A = T(3.0) * cu;
        const T B = T(4.5) * cu * cu;
        const T fq = feq_of<T, QUASI>(q, rho, (A + B) - c15);
        const T fo = feq_of<T, QUASI>(o, rho, (B - A) - c15);
        g[q] = g[q] + inv_tau * (fq - g[q]);
        g[o] = g[o] + inv_tau * (fo - g[o]);
    }
    return status_of<T, QUASI>(rho, usq, guard_sq);
}

// feq - g in the reference's order (collision.py:94-121, 244-246) for
// direction q and, with it, opp(q) (they share c.u, 3 cu and 4.5 cu cu):
// the deviations the MRT operator is applied to.  q with opp(q) < q is
// done by its partner.
template <class T, int QUASI>
__device__ __forceinline__ void mrt_dev_at(int q, const T (&g)[Q], T (&d)[Q], T rho,
                                           const T (&u)[3], T c15) {
    if (q == 0) {
        d[0] = feq_of<T, QUASI>(0, rho, (T(3.0) * T(0) + T(4.5) * T(0) * T(0)) - c15) - g[0];
        return;
    }
    if (opp(q) < q) return;
    const int o = opp(q);
    T cu = T(0);
    bool first = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int e = e_axis(q, a);
        if (e == 0) continue;
        const T term = e > 0 ? u[a] : -u[a];
        cu = first ? term : cu + term;
        first = false;
    }
    const T A = T(3.0) * cu;
    const T B = T(4.5) * cu * cu;
    d[q] = feq_of<T, QUASI>(q, rho, (A + B) - c15) - g[q];
    d[o] = feq_of<T, QUASI>(o, rho, (B - A) - c15) - g[o];
}

// all 19 deviations; returns the status word
template <class T, int QUASI>
__device__ __forceinline__ uint32_t mrt_deviations(const T (&g)[Q], T (&d)[Q], T guard_sq) {
    T rho, u[3];
    moments<T, QUASI>(g, rho, u);
    const T usq = speed_sq(u);
    const T c15 = T(1.5) * usq;
#pragma unroll
    for (int q = 0; q < Q; ++q) mrt_dev_at<T, QUASI>(q, g, d, rho, u, c15);
    return status_of<T, QUASI>(rho, usq, guard_sq);
}

// MRT collide in place: g <- g + A (feq - g) with the velocity-space operator
// A = M^-1 S M (collision.py:206-247), A row-major in op[19*19].  Rows are
// accumulated from 0 in column order like apply_operator (collision.py:216-
// 231).  The reference skips exact-zero coefficients; adding their c * d = 0
// terms instead leaves every finite result bit-identical (x + 0 = x), so the
// kernel runs the dense 19 x 19 product with coefficients read straight from
// the kernel-parameter constant bank (compile-time offsets after unrolling).
//
// grouped (default operator, checked on the host per launch): op holds, per
// column j, only the distinct values of A[.][j] (mrt_pattern.cuh), and each
// distinct product c * d[j] is computed once and added to every row that
// holds c -- the same rounded product in the same row order, so the result
// equals the dense product bit for bit (up to the sign of an all-zero row
// sum: the first term starts the row instead of 0 + term).  209 instead of
// 361 multiplies, and 19 independent row chains.
// fp32 grouped products in pairs: one packed FMUL2 (sm_100a mul.rn.f32x2,
// IEEE round-to-nearest per lane, so bit-identical to two FMULs) for two
// distinct values of a column; the row sums stay scalar FADDs, which ptxas
// does not contract with a packed product.  Columns start at even offsets
// of the operator table (mrt_offset_even) so each pair is one 8-byte load.
// 0: scalar, 1: packed products (FMUL2), 2: packed products and row sums
// (FFMA2 + FADD2, below).  The block-store kernel runs 2 (256^3 channel
// 0.623 -> 0.586 ms at 32 warps/SM); the compact kernels run 1 (the
// node-parallel step holds two nodes per thread and loses with 2:
// porosity 0.2 0.1345 -> 0.141 ms) (scripts/exp/exp71.sh)
#ifndef TLBM_MRT_PACKED
#define TLBM_MRT_PACKED 2
#endif
#ifndef TLBM_MRT_PACKED_COMPACT
#define TLBM_MRT_PACKED_COMPACT 1
#endif
__host__ __device__ constexpr int mrt_offset_even(int j) {
    int o = 0;
    for (int c = 0; c < j; ++c) o += (mrt_count(c) + 1) & ~1;
    return o;
}
// where column j's distinct values start in the kernel's operator table
template <class T, int PACK>
__host__ __device__ constexpr int mrt_table_offset(int j) {
    return (sizeof(T) == 4 && PACK == 1) ? mrt_offset_even(j) : mrt_offset(j);
}
__device__ __forceinline__ void mul2_bcast(const float *c, float d, float &r0, float &r1) {
    unsigned long long cc, dd, rr;
    asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c[0]), "f"(c[1]));
    asm("mov.b64 %0, {%1, %1};" : "=l"(dd) : "f"(d));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(cc), "l"(dd));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r0), "=f"(r1) : "l"(rr));
}

// TLBM_MRT_PACKED 2: the row sums too, two rows per FADD2 (add.rn.f32x2,
// bit-identical to two FADDs).  Rows are paired (mrt_pair_row); for each
// column the pairs' product pairs (c_a d, c_b d) come from one packed
// multiply per distinct (value, value) combination (mrt_combo_group).  The
// multiply is fma.rn.f32x2(c, d, -0): c*d + (-0) rounds the exact product
// once, so it equals mul.rn bit for bit (an exact +0 product stays +0), and
// ptxas cannot contract it into the following FADD2 -- it does contract
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under -fmad=false.  The -0
// pair is loaded from global memory (tlbm_neg_zero2), opaque to ptxas and in
// an ordinary register, so every coefficient pair stays a uniform-register
// operand (LDCU.128, two pairs per load); from the kernel parameters it
// would be uniform too and push the coefficients into LDC.64 + registers.
static __device__ unsigned long long tlbm_neg_zero2 = 0x8000000080000000ull;
__device__ __forceinline__ unsigned long long fma2_bcast_zero(const float *c, float d,
                                                              unsigned long long z) {
    unsigned long long cc, dd, rr;
    asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c[0]), "f"(c[1]));
    asm("mov.b64 %0, {%1, %1};" : "=l"(dd) : "f"(d));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rr) : "l"(cc), "l"(dd), "l"(z));
    return rr;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float lane_of(unsigned long long v, int h) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return h ? hi : lo;
}

__device__ __forceinline__ void mrt_product_paired(float (&g)[Q], const float (&d)[Q],
                                                   const float *op) {
    const unsigned long long z = tlbm_neg_zero2;
    unsigned long long acc[kMrtPairs];
    float acc_s = 0.f;
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        unsigned long long pr[kMrtMaxCombos];
#pragma unroll
        for (int c = 0; c < kMrtMaxCombos; ++c)
            if (c < mrt_ncombo(j))
                pr[c] = fma2_bcast_zero(op + 2 * (mrt_combo_offset(j) + c), d[j], z);
#pragma unroll
        for (int p = 0; p < kMrtPairs; ++p)
            acc[p] = j == 0 ? pr[mrt_pair_combo(p, j)] : add2(acc[p], pr[mrt_pair_combo(p, j)]);
        constexpr int kNone = -1;
        const float ps = mrt_single_lane(j) != kNone
                             ? lane_of(pr[mrt_single_lane(j) >> 1], mrt_single_lane(j) & 1)
                             : op[mrt_single_offset(j)] * d[j];
        acc_s = j == 0 ? ps : acc_s + ps;
    }
#pragma unroll
    for (int p = 0; p < kMrtPairs; ++p) {
        g[mrt_pair_row(p, 0)] = g[mrt_pair_row(p, 0)] + lane_of(acc[p], 0);
        g[mrt_pair_row(p, 1)] = g[mrt_pair_row(p, 1)] + lane_of(acc[p], 1);
    }
    g[kMrtSingleRow] = g[kMrtSingleRow] + acc_s;
}

// PACK: the fp32 packing (TLBM_MRT_PACKED); the operator table's layout
// follows it (fill_params)
template <class T, int QUASI, int PACK = 0>
__device__ __forceinline__ uint32_t collide_mrt(T (&g)[Q], const T *op, T guard_sq,
                                                bool grouped = false) {
    // (computing each column's deviations right before its products instead
    // of all 19 up front frees registers but ran 1.7% / 1.0% slower in
    // fp64 / fp32 on the 256^3 channel, scripts/exp/exp74.sh)
    if constexpr (sizeof(T) == 4 && PACK == 2) {
        if (TLBM_MRT_GROUPED && grouped) {
            // the status word before the deviations -- the same operations,
            // scheduled by ptxas into 0.568 vs 0.586 ms on the 256^3
            // channel (fp64's grouped product the other way round: 1.010 vs
            // 0.986 ms; scripts/exp/exp75.sh)
            T rho, u[3];
            moments<T, QUASI>(g, rho, u);
            const T usq = speed_sq(u);
            const T c15 = T(1.5) * usq;
            const uint32_t st = status_of<T, QUASI>(rho, usq, guard_sq);
            T d[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) mrt_dev_at<T, QUASI>(q, g, d, rho, u, c15);
            mrt_product_paired(reinterpret_cast<float (&)[Q]>(g),
                               reinterpret_cast<const float (&)[Q]>(d),
                               reinterpret_cast<const float *>(op));
            return st;
        }
    }
    T d[Q];
    const uint32_t st = mrt_deviations<T, QUASI>(g, d, guard_sq);
    if (TLBM_MRT_GROUPED && grouped) {
        T acc[Q];
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            T prod[kMrtMaxPerColumn];
            constexpr bool kPacked = sizeof(T) == 4 && PACK == 1;
            const int o = mrt_table_offset<T, PACK>(j);
#pragma unroll
            for (int k = 0; k < kMrtMaxPerColumn; ++k) {
                if (k >= mrt_count(j)) continue;
                if constexpr (kPacked) {
                    if (k & 1) continue;
                    if (k + 1 < mrt_count(j)) {
                        mul2_bcast(reinterpret_cast<const float *>(op + o + k), float(d[j]),
                                   reinterpret_cast<float &>(prod[k]),
                                   reinterpret_cast<float &>(prod[k + 1]));
                        continue;
                    }
                }
                prod[k] = op[o + k] * d[j];
            }
#pragma unroll
            for (int i = 0; i < Q; ++i)
                acc[i] = j == 0 ? prod[mrt_group(i, j)] : acc[i] + prod[mrt_group(i, j)];
        }
#pragma unroll
        for (int i = 0; i < Q; ++i) g[i] = g[i] + acc[i];
        return st;
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        T acc = T(0);
#pragma unroll
        for (int j = 0; j < Q; ++j) acc = acc + op[i * Q + j] * d[j];
        g[i] = g[i] + acc;
    }
    return st;
}

// ---- Zou-He (boundaries.py:53-92 closures, 132-195 arithmetic) -----------
// FACE = 2*axis + (0 low face, inward sign +1 | 1 high face, sign -1)
__host__ __device__ constexpr int face_axis(int face) { return face >> 1; }
__host__ __device__ constexpr int face_sign(int face) { return (face & 1) ? -1 : 1; }
__host__ __device__ constexpr int c_dot_n(int q, int face) {
    return e_axis(q, face_axis(face)) * face_sign(face);
}
// the unknown axis direction (c = n)
__host__ __device__ constexpr int face_axis_dir(int face) {
    return face == 0 ? 1 : face == 1 ? 3 : face == 2 ? 2 : face == 3 ? 4 : face == 4 ? 5 : 6;
}
// transverse axis of an unknown diagonal
__host__ __device__ constexpr int diag_tau(int q, int face) {
    return (face_axis(face) != 0 && ex(q) != 0) ? 0
         : (face_axis(face) != 1 && ey(q) != 0) ? 1 : 2;
}

// ordered sum over the directions with c.n == cn and, if tau >= 0,
// c_tau == sgn, in index order (boundaries.py:132-136)
template <class T, int FACE>
__device__ __forceinline__ T ordered_sum(const T (&g)[Q], int cn, int tau, int sgn) {
    T acc = T(0);
    bool first = true;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (c_dot_n(q, FACE) == cn && (tau < 0 || e_axis(q, tau) == sgn)) {
            if (first) { acc = g[q]; first = false; }
            else acc = acc + g[q];
        }
    }
    return acc;
}

// _apply_closure (boundaries.py:179-195)
template <class T, int FACE>
__device__ __forceinline__ void zh_close(T (&g)[Q], const T (&j)[3]) {
    constexpr int AX = face_axis(FACE);
    constexpr int TQ = face_axis_dir(FACE);
    const T third = T(1.0 / 3.0), sixth = T(1.0 / 6.0), half = T(0.5);
    T jn = T(face_sign(FACE)) * j[AX];
    g[TQ] = g[opp(TQ)] + third * jn;
    T ntau[3];
#pragma unroll
    for (int tau = 0; tau < 3; ++tau) {
        if (tau == AX) continue;
        ntau[tau] = half * (ordered_sum<T, FACE>(g, 0, tau, 1) - ordered_sum<T, FACE>(g, 0, tau, -1))
                  - third * j[tau];
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (c_dot_n(q, FACE) != 1 || q == TQ) continue;
        const int tau = diag_tau(q, FACE);
        const T s = T(e_axis(q, tau));
        g[q] = g[opp(q)] + sixth * (jn + s * j[tau]) - s * ntau[tau];
    }
}

// zou_he_velocity (boundaries.py:139-157)
template <class T, int QUASI, int FACE>
__device__ __forceinline__ void zh_velocity(T (&g)[Q], const double (&u_in)[3]) {
    constexpr int AX = face_axis(FACE);
    T u[3] = {T(u_in[0]), T(u_in[1]), T(u_in[2])};
    T j[3];
    if (QUASI) {
        T un = T(face_sign(FACE)) * u[AX];
        T k0 = ordered_sum<T, FACE>(g, 0, -1, 0);
        T km = ordered_sum<T, FACE>(g, -1, -1, 0);
        T rho = (k0 + T(2.0) * km) / (T(1.0) - un);
#pragma unroll
        for (int a = 0; a < 3; ++a) j[a] = u[a] * rho;
    } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) j[a] = u[a];
    }
    zh_close<T, FACE>(g, j);
}

// zou_he_pressure (boundaries.py:160-176)
template <class T, int FACE>
__device__ __forceinline__ void zh_pressure(T (&g)[Q], double rho0_in) {
    constexpr int AX = face_axis(FACE);
    T rho0 = T(rho0_in);
    T k0 = ordered_sum<T, FACE>(g, 0, -1, 0);
    T km = ordered_sum<T, FACE>(g, -1, -1, 0);
    T jn = rho0 - (k0 + T(2.0) * km);
    T j[3] = {T(0), T(0), T(0)};
    j[AX] = T(face_sign(FACE)) * jn;
    zh_close<T, FACE>(g, j);
}

template <class T, int QUASI>
__device__ __forceinline__ void zou_he_inline(T (&g)[Q], int tag, int face,
                                           const double (&u_in)[3], double rho0) {
    if (tag == INLET) {
        switch (face) {
            case 0: zh_velocity<T, QUASI, 0>(g, u_in); break;
            case 1: zh_velocity<T, QUASI, 1>(g, u_in); break;
            case 2: zh_velocity<T, QUASI, 2>(g, u_in); break;
            case 3: zh_velocity<T, QUASI, 3>(g, u_in); break;
            case 4: zh_velocity<T, QUASI, 4>(g, u_in); break;
            default: zh_velocity<T, QUASI, 5>(g, u_in); break;
        }
    } else {
        switch (face) {
            case 0: zh_pressure<T, 0>(g, rho0); break;
            case 1: zh_pressure<T, 1>(g, rho0); break;
            case 2: zh_pressure<T, 2>(g, rho0); break;
            case 3: zh_pressure<T, 3>(g, rho0); break;
            case 4: zh_pressure<T, 4>(g, rho0); break;
            default: zh_pressure<T, 5>(g, rho0); break;
        }
    }
}

// Out-of-line closure for the step kernel: inlet/outlet nodes are rare, so
// the 12 face x kind variants live in one called function working on a
// stack copy; the hot FLUID path keeps g[] in registers and its register
// budget free of the closure code.
template <class T, int QUASI>
__device__ __noinline__ void zou_he_call(T *g, int tag, int face, double ux, double uy,
                                         double uz, double rho0) {
    T r[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) r[q] = g[q];
    const double u_in[3] = {ux, uy, uz};
    zou_he_inline<T, QUASI>(r, tag, face, u_in, rho0);
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] = r[q];
}

template <class T, int QUASI>
__device__ __forceinline__ void zou_he(T (&g)[Q], int tag, int face, const double (&u_in)[3],
                                    double rho0) {
    T tmp[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) tmp[q] = g[q];
    zou_he_call<T, QUASI>(tmp, tag, face, u_in[0], u_in[1], u_in[2], rho0);
#pragma unroll
    for (int q = 0; q < Q; ++q) g[q] = tmp[q];
}

}  // namespace tlbm
