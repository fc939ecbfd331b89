/* Matrix-free P1 operator applies on the structured meshes -- ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the element sums the reference assembles into CSR and multiplies
 * (fem.py:233-276; oracle/p1.py ``Kuu`` / ``Kaa``), for the config-5 check at sizes where the
 * assembled oracle matrix does not fit ("a matrix-free CPU restatement ... validated
 * against the assembled oracle at the overlapping sizes").  Same element loops, geometry and
 * coefficients as oracle/p1.py:
 *
 *   Kuu x = sum_e a(abar_e) |T_e| E B_e^T D1 B_e x_e,          a = (1 - abar)^2 + k_ell
 *   Kaa x = sum_e react_e (1/(d+1)^2) 1 1^T x_e + 2 (Gc/c_w) ell |T_e| G_e^T G_e x_e,
 *           react_e = (1/2 a'' q_e + (Gc/c_w) w''/ell) |T_e|,  q_e = E eps(u_e)^T D1 eps(u_e)
 *
 * Meshes (oracle/meshgen.py): 2D grid vertex (i, j) = i*(ny+1)+j at linspace coordinates, crossed
 * centres appended as Vc + I*ny + J, union-jack / right / crossed cell splits; 3D Kuhn hexes (the
 * six axis-order paths from v000 to v111), vertex (i, j, k) = (i*(ny+1)+j)*(nz+1)+k.  Element node
 * order does not change a symmetric element matrix, so each simplex takes |det|.
 *
 * Threads: cell rows (2D) / cell slabs (3D) in two colour passes (even, then odd) so no two
 * threads scatter into the same vertex; the result is independent of the thread count.
 * Built by oracle/build_oracle.py into oracle/_c/libpf_oracle_mf.so (gcc -O2 -fopenmp).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

enum { UNION_JACK = 0, RIGHT = 1, CROSSED = 2 };
enum { PLANE_STRESS = 0, PLANE_STRAIN = 1 };

typedef struct {
    double E, nu, Gc, ell, k_ell;
    int model;   /* 0 AT1, 1 AT2 */
    int regime;  /* 2D: 0 plane stress, 1 plane strain; 3D ignored */
} mf_mat;

static double lin(double lo, double hi, long n, long i) { /* numpy.linspace(lo, hi, n + 1)[i] */
    if (i == n) return hi;
    return lo + (double)i * ((hi - lo) / (double)n);
}

static void d1_2d(const mf_mat* m, double D[3][3]) {
    const double nu = m->nu;
    memset(D, 0, sizeof(double) * 9);
    if (m->regime == PLANE_STRESS) {
        const double s = 1.0 / (1.0 - nu * nu);
        D[0][0] = D[1][1] = s;
        D[0][1] = D[1][0] = s * nu;
        D[2][2] = s * 0.5 * (1.0 - nu);
    } else {
        const double s = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu));
        D[0][0] = D[1][1] = s * (1.0 - nu);
        D[0][1] = D[1][0] = s * nu;
        D[2][2] = s * 0.5 * (1.0 - 2.0 * nu);
    }
}

/* one triangle: op 0 = Kuu (x: 2 dofs per node, uses alpha), op 1 = Kaa (x: 1 dof, uses u) */
static void tri(int op, const mf_mat* m, double D[3][3], const double* X, const double* Y, const long* v,
                const double* alpha, const double* u, const double* x, double* y) {
    const double det = (X[1] - X[0]) * (Y[2] - Y[0]) - (Y[1] - Y[0]) * (X[2] - X[0]);
    const double ad = fabs(det);
    const double b[3] = {(Y[1] - Y[2]) / det, (Y[2] - Y[0]) / det, (Y[0] - Y[1]) / det};
    const double c[3] = {(X[2] - X[1]) / det, (X[0] - X[2]) / det, (X[1] - X[0]) / det};
    const double vol = 0.5 * ad;
    if (op == 0) {
        const double ab = (alpha[v[0]] + alpha[v[1]] + alpha[v[2]]) / 3.0;
        const double a = (1.0 - ab) * (1.0 - ab) + m->k_ell;
        double e[3] = {0, 0, 0};
        for (int n = 0; n < 3; ++n) {
            const double x0 = x[2 * v[n]], x1 = x[2 * v[n] + 1];
            e[0] += b[n] * x0;
            e[1] += c[n] * x1;
            e[2] += c[n] * x0 + b[n] * x1;
        }
        double s[3];
        for (int r = 0; r < 3; ++r) s[r] = D[r][0] * e[0] + D[r][1] * e[1] + D[r][2] * e[2];
        const double f = a * vol * m->E;
        for (int n = 0; n < 3; ++n) {
            y[2 * v[n]] += f * (b[n] * s[0] + c[n] * s[2]);
            y[2 * v[n] + 1] += f * (c[n] * s[1] + b[n] * s[2]);
        }
    } else {
        double e[3] = {0, 0, 0};
        for (int n = 0; n < 3; ++n) {
            const double u0 = u[2 * v[n]], u1 = u[2 * v[n] + 1];
            e[0] += b[n] * u0;
            e[1] += c[n] * u1;
            e[2] += c[n] * u0 + b[n] * u1;
        }
        double q = 0.0;
        for (int r = 0; r < 3; ++r) q += e[r] * (D[r][0] * e[0] + D[r][1] * e[1] + D[r][2] * e[2]);
        q *= m->E;
        const double cw = m->model == 0 ? 8.0 / 3.0 : 2.0, wpp = m->model == 0 ? 0.0 : 2.0;
        const double kc = m->Gc / cw;
        const double react = (0.5 * 2.0 * q + kc * wpp / m->ell) * vol / 9.0;
        const double sx = x[v[0]] + x[v[1]] + x[v[2]];
        const double gx = b[0] * x[v[0]] + b[1] * x[v[1]] + b[2] * x[v[2]];
        const double gy = c[0] * x[v[0]] + c[1] * x[v[1]] + c[2] * x[v[2]];
        const double f = 2.0 * kc * m->ell * vol;
        for (int n = 0; n < 3; ++n) y[v[n]] += react * sx + f * (b[n] * gx + c[n] * gy);
    }
}

static void cell_row_2d(int op, int pattern, long nx, long ny, double lx, double ly, const mf_mat* m,
                        double D[3][3], long I, const double* alpha, const double* u, const double* x, double* y) {
    const long nv = ny + 1, vc = (nx + 1) * (ny + 1);
    const double x0 = lin(0.0, lx, nx, I), x1 = lin(0.0, lx, nx, I + 1);
    for (long J = 0; J < ny; ++J) {
        const double y0 = lin(0.0, ly, ny, J), y1 = lin(0.0, ly, ny, J + 1);
        const long a = I * nv + J, b = (I + 1) * nv + J, c = (I + 1) * nv + J + 1, d = I * nv + J + 1;
        /* corner coordinates by local slot a, b, c, d */
        const double cx[4] = {x0, x1, x1, x0}, cyy[4] = {y0, y0, y1, y1};
        const long cv[4] = {a, b, c, d};
        long t[4][3];
        int nt = 2;
        if (pattern == CROSSED) {
            nt = 4;
        } else if (pattern == RIGHT || ((I + J) % 2 == 0)) {
            long t0[3] = {0, 1, 2}, t1[3] = {0, 2, 3};
            memcpy(t[0], t0, sizeof t0);
            memcpy(t[1], t1, sizeof t1);
        } else {
            long t0[3] = {0, 1, 3}, t1[3] = {1, 2, 3};
            memcpy(t[0], t0, sizeof t0);
            memcpy(t[1], t1, sizeof t1);
        }
        if (pattern == CROSSED) {
            const long ctr = vc + I * ny + J;
            const double xc = 0.5 * (x0 + x1), yc = 0.5 * (y0 + y1);
            const int pr[4][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}};
            for (int k = 0; k < 4; ++k) {
                const long v[3] = {cv[pr[k][0]], cv[pr[k][1]], ctr};
                const double X[3] = {cx[pr[k][0]], cx[pr[k][1]], xc}, Y[3] = {cyy[pr[k][0]], cyy[pr[k][1]], yc};
                tri(op, m, D, X, Y, v, alpha, u, x, y);
            }
        } else {
            for (int k = 0; k < nt; ++k) {
                const long v[3] = {cv[t[k][0]], cv[t[k][1]], cv[t[k][2]]};
                const double X[3] = {cx[t[k][0]], cx[t[k][1]], cx[t[k][2]]};
                const double Y[3] = {cyy[t[k][0]], cyy[t[k][1]], cyy[t[k][2]]};
                tri(op, m, D, X, Y, v, alpha, u, x, y);
            }
        }
    }
}

/* y = K x (y overwritten); op 0 = Kuu (alpha, x: 2 per vertex), op 1 = Kaa (u, x: 1 per vertex) */
int pf_oracle_mf_2d(int op, int pattern, long nx, long ny, double lx, double ly, const mf_mat* m,
                    const double* alpha, const double* u, const double* x, double* y, int nthreads) {
    const long nvert = (nx + 1) * (ny + 1) + (pattern == CROSSED ? nx * ny : 0);
    memset(y, 0, sizeof(double) * (size_t)nvert * (op == 0 ? 2 : 1));
    double D[3][3];
    d1_2d(m, D);
    for (int colour = 0; colour < 2; ++colour) {
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
        for (long I = colour; I < nx; I += 2) cell_row_2d(op, pattern, nx, ny, lx, ly, m, D, I, alpha, u, x, y);
    }
    return 0;
}

/* ---- 3D Kuhn ---- */
static void tet(int op, const mf_mat* m, const double P[4][3], const long* v, const double* alpha,
                const double* u, const double* x, double* y) {
    double J[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) J[r][c] = P[c + 1][r] - P[0][r]; /* columns p_{c+1} - p_0 */
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    double inv[3][3]; /* inv(J) by the adjugate */
    inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    double G[4][3]; /* gradient of lambda_n: n >= 1 -> row n-1 of inv(J) */
    for (int n = 1; n < 4; ++n)
        for (int a = 0; a < 3; ++a) G[n][a] = inv[n - 1][a];
    for (int a = 0; a < 3; ++a) G[0][a] = -(G[1][a] + G[2][a] + G[3][a]);
    const double vol = fabs(det) / 6.0;
    const double nu = m->nu, lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), mu = 1.0 / (2.0 * (1.0 + nu));
    const double* f = op == 0 ? x : u;
    double e[6] = {0, 0, 0, 0, 0, 0};
    for (int n = 0; n < 4; ++n) {
        const double a0 = f[3 * v[n]], a1 = f[3 * v[n] + 1], a2 = f[3 * v[n] + 2];
        const double gx = G[n][0], gy = G[n][1], gz = G[n][2];
        e[0] += gx * a0;
        e[1] += gy * a1;
        e[2] += gz * a2;
        e[3] += gz * a1 + gy * a2;
        e[4] += gz * a0 + gx * a2;
        e[5] += gy * a0 + gx * a1;
    }
    const double tr = e[0] + e[1] + e[2];
    const double s[6] = {lam * tr + 2 * mu * e[0], lam * tr + 2 * mu * e[1], lam * tr + 2 * mu * e[2],
                         mu * e[3], mu * e[4], mu * e[5]};
    if (op == 0) {
        const double ab = 0.25 * (alpha[v[0]] + alpha[v[1]] + alpha[v[2]] + alpha[v[3]]);
        const double a = (1.0 - ab) * (1.0 - ab) + m->k_ell;
        const double fc = a * vol * m->E;
        for (int n = 0; n < 4; ++n) {
            const double gx = G[n][0], gy = G[n][1], gz = G[n][2];
            y[3 * v[n]] += fc * (gx * s[0] + gz * s[4] + gy * s[5]);
            y[3 * v[n] + 1] += fc * (gy * s[1] + gz * s[3] + gx * s[5]);
            y[3 * v[n] + 2] += fc * (gz * s[2] + gy * s[3] + gx * s[4]);
        }
    } else {
        double q = 0.0;
        for (int r = 0; r < 6; ++r) q += e[r] * s[r];
        q *= m->E;
        const double cw = m->model == 0 ? 8.0 / 3.0 : 2.0, wpp = m->model == 0 ? 0.0 : 2.0;
        const double kc = m->Gc / cw;
        const double react = (0.5 * 2.0 * q + kc * wpp / m->ell) * vol / 16.0;
        double sx = 0.0, g[3] = {0, 0, 0};
        for (int n = 0; n < 4; ++n) {
            sx += x[v[n]];
            for (int a = 0; a < 3; ++a) g[a] += G[n][a] * x[v[n]];
        }
        const double fc = 2.0 * kc * m->ell * vol;
        for (int n = 0; n < 4; ++n) y[v[n]] += react * sx + fc * (G[n][0] * g[0] + G[n][1] * g[1] + G[n][2] * g[2]);
    }
}

static const int kPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

int pf_oracle_mf_3d(int op, long nx, long ny, long nz, double lx, double ly, double lz, const mf_mat* m,
                    const double* alpha, const double* u, const double* x, double* y, int nthreads) {
    const long nvert = (nx + 1) * (ny + 1) * (nz + 1);
    memset(y, 0, sizeof(double) * (size_t)nvert * (op == 0 ? 3 : 1));
    const long n[3] = {nx, ny, nz};
    const double L[3] = {lx, ly, lz};
    for (int colour = 0; colour < 2; ++colour) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
        for (long I = colour; I < nx; I += 2) {
            for (long Jc = 0; Jc < ny; ++Jc)
                for (long Kc = 0; Kc < nz; ++Kc) {
                    const long base[3] = {I, Jc, Kc};
                    for (int t = 0; t < 6; ++t) {
                        long cur[3] = {0, 0, 0};
                        long v[4];
                        double P[4][3];
                        for (int p = 0; p < 4; ++p) {
                            if (p > 0) cur[kPerm[t][p - 1]] = 1;
                            long id[3];
                            for (int a = 0; a < 3; ++a) {
                                id[a] = base[a] + cur[a];
                                P[p][a] = lin(0.0, L[a], n[a], id[a]);
                            }
                            v[p] = (id[0] * (ny + 1) + id[1]) * (nz + 1) + id[2];
                        }
                        tet(op, m, P, v, alpha, u, x, y);
                    }
                }
        }
    }
    return 0;
}
