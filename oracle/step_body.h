/* Generic body of the oracle step, included once per REAL type by
 * tlbm_oracle.c (REAL = double | float, SFX = f64 | f32).  TEST
 * INFRASTRUCTURE ONLY -- see tlbm_oracle.c. */
#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)

/* collision.py:46-130 for one node, in the reference's operation order;
 * writes the post-collision populations into out and returns the status
 * bits (1 divergence, 2 guard). */
static int CAT(collide, SFX)(const REAL *g, REAL *out, int quasi, REAL inv_tau,
                             double u_guard) {
    REAL rho = g[0];
    for (int q = 1; q < 19; ++q) rho += g[q];
    REAL j[3];
    for (int a = 0; a < 3; ++a) {
        REAL acc = (REAL)0;
        for (int q = 0; q < 19; ++q) {
            if (EV[q][a] == 1) acc += g[q];
            else if (EV[q][a] == -1) acc -= g[q];
        }
        j[a] = acc;
    }
    int st = 0;
    if (rho != rho || (quasi && !(rho > (REAL)0))) st |= 1;
    REAL u[3];
    for (int a = 0; a < 3; ++a) u[a] = quasi ? j[a] / rho : j[a];
    REAL usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    if (u_guard > 0 && usq > (REAL)(u_guard * u_guard)) st |= 2;
    for (int q = 0; q < 19; ++q) {
        REAL cu = (REAL)0;
        for (int a = 0; a < 3; ++a) {
            if (EV[q][a] > 0) cu += u[a];
            else if (EV[q][a] < 0) cu += -u[a];
        }
        REAL br = (REAL)3.0 * cu + (REAL)4.5 * cu * cu - (REAL)1.5 * usq;
        REAL w = (REAL)(q == 0 ? 1.0 / 3.0 : (q < 7 ? 1.0 / 18.0 : 1.0 / 36.0));
        REAL feq = quasi ? w * (rho * ((REAL)1.0 + br)) : w * (rho + br);
        out[q] = g[q] + inv_tau * (feq - g[q]);
    }
    return st;
}

/* collide_mrt (collision.py:216-247): g + apply_operator(op, feq - g), the
 * operator rows accumulated from 0 in column order, zero coefficients
 * skipped. */
static int CAT(collide_mrt, SFX)(const REAL *g, REAL *out, int quasi, const REAL *op,
                                 double u_guard) {
    REAL rho = g[0];
    for (int q = 1; q < 19; ++q) rho += g[q];
    REAL j[3];
    for (int a = 0; a < 3; ++a) {
        REAL acc = (REAL)0;
        for (int q = 0; q < 19; ++q) {
            if (EV[q][a] == 1) acc += g[q];
            else if (EV[q][a] == -1) acc -= g[q];
        }
        j[a] = acc;
    }
    int st = 0;
    if (rho != rho || (quasi && !(rho > (REAL)0))) st |= 1;
    REAL u[3];
    for (int a = 0; a < 3; ++a) u[a] = quasi ? j[a] / rho : j[a];
    REAL usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    if (u_guard > 0 && usq > (REAL)(u_guard * u_guard)) st |= 2;
    REAL delta[19];
    for (int q = 0; q < 19; ++q) {
        REAL cu = (REAL)0;
        for (int a = 0; a < 3; ++a) {
            if (EV[q][a] > 0) cu += u[a];
            else if (EV[q][a] < 0) cu += -u[a];
        }
        REAL br = (REAL)3.0 * cu + (REAL)4.5 * cu * cu - (REAL)1.5 * usq;
        REAL w = (REAL)(q == 0 ? 1.0 / 3.0 : (q < 7 ? 1.0 / 18.0 : 1.0 / 36.0));
        REAL feq = quasi ? w * (rho * ((REAL)1.0 + br)) : w * (rho + br);
        delta[q] = feq - g[q];
    }
    for (int i = 0; i < 19; ++i) {
        REAL acc = (REAL)0;
        for (int k = 0; k < 19; ++k) {
            REAL c = op[i * 19 + k];
            if (c != (REAL)0) acc += c * delta[k];
        }
        out[i] = g[i] + acc;
    }
    return st;
}

static REAL CAT(osum, SFX)(const REAL *g, const int *d, int n) {
    REAL acc = g[d[0]];
    for (int i = 1; i < n; ++i) acc += g[d[i]];
    return acc;
}

/* boundaries.py:179-195 */
static void CAT(close, SFX)(REAL *g, const face_t *c, const REAL *j) {
    const REAL third = (REAL)(1.0 / 3.0), sixth = (REAL)(1.0 / 6.0);
    REAL jn = (REAL)c->sign * j[c->axis];
    g[c->t] = g[c->t_opp] + third * jn;
    REAL ntau[3] = {0, 0, 0};
    for (int k = 0; k < 2; ++k) {
        int tau = c->taus[k];
        ntau[tau] = (REAL)0.5 * (CAT(osum, SFX)(g, c->plus[k], c->np[k])
                                 - CAT(osum, SFX)(g, c->minus[k], c->nm[k]))
                    - third * j[tau];
    }
    for (int i = 0; i < c->ndiag; ++i) {
        REAL s = (REAL)c->dsig[i];
        g[c->dq[i]] = g[c->dqo[i]] + sixth * (jn + s * j[c->dtau[i]])
                      - s * ntau[c->dtau[i]];
    }
}

/* boundaries.py:139-157 */
static void CAT(zh_velocity, SFX)(REAL *g, const face_t *c, const double *u_in,
                                  int quasi) {
    REAL u[3] = {(REAL)u_in[0], (REAL)u_in[1], (REAL)u_in[2]};
    REAL un = (REAL)c->sign * u[c->axis];
    REAL k0 = CAT(osum, SFX)(g, c->k0, c->nk0);
    REAL km = CAT(osum, SFX)(g, c->km, c->nkm);
    REAL j[3];
    if (quasi) {
        REAL rho = (k0 + (REAL)2.0 * km) / ((REAL)1.0 - un);
        for (int a = 0; a < 3; ++a) j[a] = u[a] * rho;
    } else {
        for (int a = 0; a < 3; ++a) j[a] = u[a];
    }
    CAT(close, SFX)(g, c, j);
}

/* boundaries.py:160-176 */
static void CAT(zh_pressure, SFX)(REAL *g, const face_t *c, double rho0_in) {
    REAL rho0 = (REAL)rho0_in;
    REAL k0 = CAT(osum, SFX)(g, c->k0, c->nk0);
    REAL km = CAT(osum, SFX)(g, c->km, c->nkm);
    REAL jn = rho0 - (k0 + (REAL)2.0 * km);
    REAL j[3] = {0, 0, 0};
    j[c->axis] = (REAL)c->sign * jn;
    CAT(close, SFX)(g, c, j);
}

/* One step: f (current copy) -> fnew (other copy).  Returns the OR of the
 * per-node status bits (1 divergence, 2 |u| guard). */
int CAT(oracle_step, SFX)(const REAL *f, REAL *fnew, const uint8_t *types,
                          const int8_t *faces, const oracle_params *p) {
    if (!faces_ready) build_faces();
    const int nx = p->nx, ny = p->ny, nz = p->nz;
    const int64_t N = (int64_t)nx * ny * nz;
    const REAL inv_tau = (REAL)(1.0 / p->tau);
    int status = 0;
#ifdef _OPENMP
    int nt = p->nthreads > 0 ? p->nthreads : omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nt) reduction(| : status)
#endif
    for (int x = 0; x < nx; ++x) {
        REAL g[19], out[19];
        for (int y = 0; y < ny; ++y) {
            for (int z = 0; z < nz; ++z) {
                const int64_t n = ((int64_t)x * ny + y) * nz + z;
                const int tag = types[n];
                if (tag == 0) continue;
                g[0] = f[n];
                for (int q = 1; q < 19; ++q) {
                    int s[3] = {x - EV[q][0], y - EV[q][1], z - EV[q][2]};
                    const int d[3] = {nx, ny, nz};
                    int ok = 1;
                    for (int a = 0; a < 3; ++a) {
                        if (s[a] < 0 || s[a] >= d[a]) {
                            if (p->periodic[a]) s[a] = (s[a] + d[a]) % d[a];
                            else ok = 0;
                        }
                    }
                    int64_t sn = 0;
                    if (ok) {
                        sn = ((int64_t)s[0] * ny + s[1]) * nz + s[2];
                        ok = types[sn] != 0;
                    }
                    g[q] = ok ? f[(int64_t)q * N + sn] : f[(int64_t)OPQ[q] * N + n];
                }
                if (tag == 2) {
                    for (int q = 0; q < 19; ++q) out[q] = g[OPQ[q]];
                } else {
                    if (tag == 3)
                        CAT(zh_velocity, SFX)(g, &FACES[faces[n]], p->inlet_u, p->quasi);
                    else if (tag == 4)
                        CAT(zh_pressure, SFX)(g, &FACES[faces[n]], p->outlet_rho);
                    if (p->mrt_op)
                        status |= CAT(collide_mrt, SFX)(g, out, p->quasi,
                                                        (const REAL *)p->mrt_op, p->u_guard);
                    else
                        status |= CAT(collide, SFX)(g, out, p->quasi, inv_tau, p->u_guard);
                }
                for (int q = 0; q < 19; ++q) fnew[(int64_t)q * N + n] = out[q];
            }
        }
    }
    return status;
}

/* Run `steps` steps ping-ponging between a and b; returns the final copy
 * index (0 = a, 1 = b) in *which and the OR of statuses.  Stops at the first
 * divergent step, reporting it in *failed_step (-1 if none). */
int CAT(oracle_run, SFX)(REAL *a, REAL *b, const uint8_t *types,
                         const int8_t *faces, const oracle_params *p, int steps,
                         int *which, int *failed_step) {
    int st_all = 0;
    REAL *cur = a, *nxt = b;
    *failed_step = -1;
    for (int i = 0; i < steps; ++i) {
        int st = CAT(oracle_step, SFX)(cur, nxt, types, faces, p);
        st_all |= st;
        REAL *t = cur; cur = nxt; nxt = t;
        if (st & 1) { *failed_step = i; break; }
    }
    *which = (cur == a) ? 0 : 1;
    return st_all;
}

#undef CAT
#undef CAT2
