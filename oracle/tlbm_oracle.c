/*
 * CPU oracle of the D3Q19 LBGK step in plain C -- TEST INFRASTRUCTURE ONLY.
 *
 * Same semantics and operation order as oracle/dense.py (SURVEY Appendix A,
 * R0-R8), i.e. the reference arithmetic of collision.py:46-130 and
 * boundaries.py:53-195 composed by the step contract of boundaries.py:1-28.
 * Compiled with -ffp-contract=off so no multiply-add is fused: results are
 * bit-identical to the numpy restatement (tests/test_oracle.py) and serve as
 * the parity reference for 1000-step GPU runs and as bench.py's CPU baseline.
 *
 * Dense layout: f[q][x][y][z] (z fastest), types[x][y][z] uint8,
 * faces[x][y][z] int8 (2*axis + (0 low | 1 high) for inlet/outlet, else -1).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int nx, ny, nz;
    int periodic[3];
    int quasi;              /* 0 incompressible, 1 quasi-compressible */
    double tau;
    double inlet_u[3];
    double outlet_rho;
    double u_guard;         /* |u| > u_guard sets flag bit 1 (0 disables) */
    int nthreads;
    const void *mrt_op;     /* NULL: LBGK; else 19x19 REAL MRT operator, row-major */
} oracle_params;

static const int EV[19][3] = {
    {0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {-1, 0, 0}, {0, -1, 0}, {0, 0, 1},
    {0, 0, -1}, {1, 1, 0}, {-1, 1, 0}, {1, -1, 0}, {-1, -1, 0}, {0, 1, 1},
    {0, 1, -1}, {0, -1, 1}, {0, -1, -1}, {1, 0, 1}, {1, 0, -1}, {-1, 0, 1},
    {-1, 0, -1}};
static const int OPQ[19] = {0, 3, 4, 1, 2, 6, 5, 10, 9, 8, 7, 14, 13, 12, 11,
                            18, 17, 16, 15};

/* Zou-He index sets of one face (boundaries.py:53-85), built at first use */
typedef struct {
    int axis, sign, t, t_opp;
    int nk0, k0[19], nkm, km[19];
    int ndiag, dq[4], dqo[4], dtau[4], dsig[4];
    int taus[2], np[2], plus[2][8], nm[2], minus[2][8];
} face_t;

static face_t FACES[6];
static int faces_ready = 0;

static void build_faces(void) {
    for (int fid = 0; fid < 6; ++fid) {
        face_t *c = &FACES[fid];
        memset(c, 0, sizeof(*c));
        c->axis = fid / 2;
        c->sign = (fid % 2 == 0) ? 1 : -1;
        for (int q = 0; q < 19; ++q) {
            int cn = EV[q][c->axis] * c->sign;
            if (cn == 0) c->k0[c->nk0++] = q;
            else if (cn == -1) c->km[c->nkm++] = q;
            else {
                int side = -1;
                for (int a = 0; a < 3; ++a)
                    if (a != c->axis && EV[q][a] != 0) { side = a; break; }
                if (side < 0) { c->t = q; c->t_opp = OPQ[q]; }
                else {
                    c->dq[c->ndiag] = q; c->dqo[c->ndiag] = OPQ[q];
                    c->dtau[c->ndiag] = side; c->dsig[c->ndiag] = EV[q][side];
                    c->ndiag++;
                }
            }
        }
        int k = 0;
        for (int tau = 0; tau < 3; ++tau) {
            if (tau == c->axis) continue;
            c->taus[k] = tau;
            for (int i = 0; i < c->nk0; ++i) {
                int q = c->k0[i];
                if (EV[q][tau] == 1) c->plus[k][c->np[k]++] = q;
                if (EV[q][tau] == -1) c->minus[k][c->nm[k]++] = q;
            }
            ++k;
        }
    }
    faces_ready = 1;
}

#define REAL double
#define SFX f64
#include "step_body.h"
#undef REAL
#undef SFX

#define REAL float
#define SFX f32
#include "step_body.h"
#undef REAL
#undef SFX

int oracle_abi_version(void) { return 1; }
