/*
 * tlsph_oracle.c -- CPU restatement of the reference TLSPH per-step kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2602_15149_b200/ links or calls
 * this file; it is the checker for the CUDA path (tests/, __graft_entry__.smoke
 * and bench.py's cpu_baseline / --impl reference arm only).
 *
 * Each function restates one kernel of the reference backend plugin
 * (/root/reference/pkg/src/solidsph/backends/reference.py, numba mirror in
 * backends/fast.py).  Semantics kept from the reference:
 *   - one writer per particle; each particle's neighbour sum runs
 *     sequentially in CSR order (the order np.add.at accumulates in,
 *     reference.py:3-6), so results are thread-count independent;
 *   - all arithmetic FP64, indices int64, tensors row-major 3x3 per particle;
 *   - kernels never raise: they return counts / first-bad indices.
 * Built with -ffp-contract=off so no FMA contraction changes rounding.
 * OpenMP parallelises the particle loop (the reference's numba prange).
 *
 * Pinned against golden vectors produced by the reference itself
 * (oracle/gen_golden.py -> tests/golden/, checked in tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define J_MIN 1.0e-6 /* core.py:45 */

typedef int64_t i64;

int orc_num_threads(void);
void orc_set_threads(int n);

#ifdef _OPENMP
#include <omp.h>
int orc_num_threads(void) { return omp_get_max_threads(); }
void orc_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
#else
int orc_num_threads(void) { return 1; }
void orc_set_threads(int n) { (void)n; }
#endif

/* ---- 3x3 helpers (fast.py:22-42) ------------------------------------- */
static double det3(const double *A) {
    return A[0] * (A[4] * A[8] - A[5] * A[7])
         - A[1] * (A[3] * A[8] - A[5] * A[6])
         + A[2] * (A[3] * A[7] - A[4] * A[6]);
}

static double inv3(const double *A, double *R) {
    double d = det3(A);
    double id = 1.0 / d;
    R[0] = (A[4] * A[8] - A[5] * A[7]) * id;
    R[1] = (A[2] * A[7] - A[1] * A[8]) * id;
    R[2] = (A[1] * A[5] - A[2] * A[4]) * id;
    R[3] = (A[5] * A[6] - A[3] * A[8]) * id;
    R[4] = (A[0] * A[8] - A[2] * A[6]) * id;
    R[5] = (A[2] * A[3] - A[0] * A[5]) * id;
    R[6] = (A[3] * A[7] - A[4] * A[6]) * id;
    R[7] = (A[1] * A[6] - A[0] * A[7]) * id;
    R[8] = (A[0] * A[4] - A[1] * A[3]) * id;
    return d;
}

static void mm3(const double *A, const double *B, double *C) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            C[3 * r + c] = A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c] + A[3 * r + 2] * B[6 + c];
}

/* Cyclic Jacobi for a symmetric 3x3, eigenvalues descending, eigenvectors in
 * the columns of Q.  Returns sweeps used (64 = no convergence).
 * Restates fast.py:45-108 (tolerance 1e-30*scale^2, skip |apq|<1e-300). */
int orc_eig3_jacobi(const double *Ain, double *w, double *Q) {
    double a[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) a[3 * r + c] = 0.5 * (Ain[3 * r + c] + Ain[3 * c + r]);
    for (int k = 0; k < 9; ++k) Q[k] = (k % 4 == 0) ? 1.0 : 0.0;
    double scale = 0.0;
    for (int k = 0; k < 9; ++k) if (fabs(a[k]) > scale) scale = fabs(a[k]);
    if (scale == 0.0) { w[0] = w[1] = w[2] = 0.0; return 0; }
    double tol = 1e-30 * scale * scale;
    int sweeps = 0;
    while (sweeps < 64) {
        double off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
        if (off <= tol) break;
        for (int p = 0; p < 2; ++p) {
            for (int q = p + 1; q < 3; ++q) {
                double apq = a[3 * p + q];
                if (fabs(apq) < 1e-300) continue;
                double theta = 0.5 * (a[3 * q + q] - a[3 * p + p]) / apq;
                double t = theta >= 0.0 ? 1.0 / (theta + sqrt(theta * theta + 1.0))
                                        : -1.0 / (-theta + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {
                    double x = a[3 * k + p], y = a[3 * k + q];
                    a[3 * k + p] = c * x - s * y;
                    a[3 * k + q] = s * x + c * y;
                }
                for (int k = 0; k < 3; ++k) {
                    double x = a[3 * p + k], y = a[3 * q + k];
                    a[3 * p + k] = c * x - s * y;
                    a[3 * q + k] = s * x + c * y;
                }
                for (int k = 0; k < 3; ++k) {
                    double x = Q[3 * k + p], y = Q[3 * k + q];
                    Q[3 * k + p] = c * x - s * y;
                    Q[3 * k + q] = s * x + c * y;
                }
            }
        }
        ++sweeps;
    }
    w[0] = a[0]; w[1] = a[4]; w[2] = a[8];
    for (int i = 0; i < 2; ++i) {
        int m = i;
        for (int j = i + 1; j < 3; ++j) if (w[j] > w[m]) m = j;
        if (m != i) {
            double tmp = w[i]; w[i] = w[m]; w[m] = tmp;
            for (int k = 0; k < 3; ++k) { tmp = Q[3 * k + i]; Q[3 * k + i] = Q[3 * k + m]; Q[3 * k + m] = tmp; }
        }
    }
    return sweeps;
}

/* ---- pair kernels ----------------------------------------------------- */

/* F_i = I + sum_j V0_j (u_j - u_i) (x) grad0_ij, gated to I when s_i <= s_l.
 * reference.py:18-29 / fast.py:111-138. */
void orc_deformation_gradient(i64 n, const i64 *indptr, const i64 *indices, const double *grad0,
                              const double *u, const double *V0, const double *s, double s_l,
                              int gated, double *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) {
        double f[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        if (!(gated && s[i] <= s_l)) {
            for (i64 k = indptr[i]; k < indptr[i + 1]; ++k) {
                i64 j = indices[k];
                double vj = V0[j];
                for (int a = 0; a < 3; ++a) {
                    double d = u[3 * j + a] - u[3 * i + a];
                    for (int b = 0; b < 3; ++b) f[3 * a + b] += (vj * d) * grad0[3 * k + b];
                }
            }
        }
        memcpy(out + 9 * i, f, sizeof f);
    }
}

/* lap_i = sum_j 2 (f_i - f_j) V0_j (r0.grad0)/|r0|^2.  reference.py:32-39. */
void orc_sph_laplacian(i64 n, const i64 *indptr, const i64 *indices, const double *grad0,
                       const double *r0, const double *r0norm, const double *V0,
                       const double *f, double *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) {
        double acc = 0.0;
        for (i64 k = indptr[i]; k < indptr[i + 1]; ++k) {
            i64 j = indices[k];
            double rdg = r0[3 * k] * grad0[3 * k] + r0[3 * k + 1] * grad0[3 * k + 1]
                       + r0[3 * k + 2] * grad0[3 * k + 2];
            acc += 2.0 * (f[i] - f[j]) * V0[j] * rdg / (r0norm[k] * r0norm[k]);
        }
        out[i] = acc;
    }
}

/* grad_i = sum_j V0_j (f_j - f_i) grad0_ij.  reference.py:42-49. */
void orc_sph_gradient(i64 n, const i64 *indptr, const i64 *indices, const double *grad0,
                      const double *V0, const double *f, double *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) {
        double g[3] = {0, 0, 0};
        for (i64 k = indptr[i]; k < indptr[i + 1]; ++k) {
            i64 j = indices[k];
            double c = V0[j] * (f[j] - f[i]);
            for (int b = 0; b < 3; ++b) g[b] += c * grad0[3 * k + b];
        }
        memcpy(out + 3 * i, g, sizeof g);
    }
}

/* TLSPH momentum with Monaghan viscosity along the corrected gradient.
 * reference.py:52-81.  Returns the count of viscosity-degenerate particles. */
i64 orc_momentum(i64 n, const i64 *indptr, const i64 *indices, const double *grad0,
                 const double *grad0r, const double *r0, const double *r0norm, const double *P,
                 const double *m0, double rho0, const double *v, double h, double c0,
                 double beta1, double beta2, const double *F, double *out) {
    int visc = (beta1 != 0.0 || beta2 != 0.0);
    double inv_rho2 = 1.0 / (rho0 * rho0);
    double eps_h2 = 0.001 * h * h;
    i64 n_bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : n_bad)
    for (i64 i = 0; i < n; ++i) {
        double Av[9] = {0};
        if (visc) {
            double Fi[9];
            memcpy(Fi, F + 9 * i, sizeof Fi);
            double d = det3(Fi);
            if (d > J_MIN) {
                inv3(Fi, Av);
                for (int q = 0; q < 9; ++q) Av[q] *= d;
            } else {
                n_bad += 1;
            }
        }
        const double *Pi = P + 9 * i;
        double acc[3] = {0, 0, 0};
        for (i64 k = indptr[i]; k < indptr[i + 1]; ++k) {
            i64 j = indices[k];
            const double *g = grad0 + 3 * k, *gr = grad0r + 3 * k, *Pj = P + 9 * j;
            double fp[3];
            for (int a = 0; a < 3; ++a) {
                double t1 = Pi[3 * a] * g[0] + Pi[3 * a + 1] * g[1] + Pi[3 * a + 2] * g[2];
                double t2 = Pj[3 * a] * gr[0] + Pj[3 * a + 1] * gr[1] + Pj[3 * a + 2] * gr[2];
                fp[a] = (t1 - t2) * inv_rho2;
            }
            if (visc) {
                double dv = (v[3 * i] - v[3 * j]) * r0[3 * k] + (v[3 * i + 1] - v[3 * j + 1]) * r0[3 * k + 1]
                          + (v[3 * i + 2] - v[3 * j + 2]) * r0[3 * k + 2];
                double G = h * dv / (r0norm[k] * r0norm[k] + eps_h2);
                double pi = (beta2 * G * G - beta1 * c0 * G) / rho0;
                for (int a = 0; a < 3; ++a)
                    fp[a] -= pi * (Av[3 * a] * g[0] + Av[3 * a + 1] * g[1] + Av[3 * a + 2] * g[2]);
            }
            for (int a = 0; a < 3; ++a) acc[a] += m0[j] * fp[a];
        }
        memcpy(out + 3 * i, acc, sizeof acc);
    }
    return n_bad;
}

/* ---- constitutive batches ------------------------------------------- */

/* St. Venant-Kirchhoff with the spectral split.  reference.py:94-116,
 * fast.py:224-284.  Returns the count of non-converged eigen solves. */
i64 orc_svk_batch(i64 n, const double *F, double lam, double mu, const double *s, int fracture,
                  double *out_S, double *out_psi, double *out_psip) {
    i64 n_noconv = 0;
#pragma omp parallel for schedule(static) reduction(+ : n_noconv)
    for (i64 i = 0; i < n; ++i) {
        const double *Fi = F + 9 * i;
        double E[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double acc = Fi[r] * Fi[c] + Fi[3 + r] * Fi[3 + c] + Fi[6 + r] * Fi[6 + c];
                E[3 * r + c] = 0.5 * (acc - (r == c ? 1.0 : 0.0));
            }
        for (int r = 0; r < 3; ++r)
            for (int c = r + 1; c < 3; ++c) {
                double m = 0.5 * (E[3 * r + c] + E[3 * c + r]);
                E[3 * r + c] = E[3 * c + r] = m;
            }
        double trE = E[0] + E[4] + E[8];
        double *S = out_S + 9 * i;
        if (!fracture) {
            double frob = 0.0;
            for (int q = 0; q < 9; ++q) { S[q] = 2.0 * mu * E[q]; frob += E[q] * E[q]; }
            S[0] += lam * trE; S[4] += lam * trE; S[8] += lam * trE;
            out_psi[i] = 0.5 * lam * trE * trE + mu * frob;
            out_psip[i] = 0.0;
            continue;
        }
        double w[3], Q[9];
        int sw = orc_eig3_jacobi(E, w, Q);
        if (sw >= 64) n_noconv += 1;
        double trp = trE > 0.0 ? trE : 0.0, trm = trE < 0.0 ? trE : 0.0;
        double psip = 0.5 * lam * trp * trp, psim = 0.5 * lam * trm * trm;
        double s2 = s[i] * s[i];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double ep = 0.0, em = 0.0;
                for (int k = 0; k < 3; ++k) {
                    double lp = w[k] > 0.0 ? w[k] : 0.0, lm = w[k] < 0.0 ? w[k] : 0.0;
                    ep += Q[3 * r + k] * lp * Q[3 * c + k];
                    em += Q[3 * r + k] * lm * Q[3 * c + k];
                }
                double sp = 2.0 * mu * ep, sm = 2.0 * mu * em;
                if (r == c) { sp += lam * trp; sm += lam * trm; }
                S[3 * r + c] = s2 * sp + sm;
            }
        for (int k = 0; k < 3; ++k) {
            double lp = w[k] > 0.0 ? w[k] : 0.0, lm = w[k] < 0.0 ? w[k] : 0.0;
            psip += mu * lp * lp;
            psim += mu * lm * lm;
        }
        out_psi[i] = s2 * psip + psim;
        out_psip[i] = psip;
    }
    return n_noconv;
}

/* Compressible neo-Hookean through b = F F^T with the volumetric split.
 * reference.py:119-148, fast.py:287-332.  Returns degenerate count. */
i64 orc_nh_batch(i64 n, const double *F, double kappa, double mu, const double *s, int fracture,
                 double *out_S, double *out_psi, double *out_psip) {
    i64 n_bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : n_bad)
    for (i64 i = 0; i < n; ++i) {
        const double *Fi = F + 9 * i;
        double *S = out_S + 9 * i;
        double J = det3(Fi);
        if (J <= J_MIN) {
            for (int q = 0; q < 9; ++q) S[q] = 0.0;
            out_psi[i] = 0.0; out_psip[i] = 0.0;
            n_bad += 1;
            continue;
        }
        double b[9], bi[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                b[3 * r + c] = Fi[3 * r] * Fi[3 * c] + Fi[3 * r + 1] * Fi[3 * c + 1] + Fi[3 * r + 2] * Fi[3 * c + 2];
        inv3(b, bi);
        double trb = b[0] + b[4] + b[8];
        double Jm23 = pow(J, -2.0 / 3.0);
        double U = 0.5 * kappa * (0.5 * (J * J - 1.0) - log(J));
        double psibar = 0.5 * mu * (Jm23 * trb - 3.0);
        double s2 = fracture ? s[i] * s[i] : 1.0;
        int tension = J >= 1.0;
        double wv = tension ? s2 : 1.0;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double svol = 0.5 * kappa * (J * J - 1.0) * bi[3 * r + c];
                double siso = Jm23 * mu * (-(trb / 3.0) * bi[3 * r + c]);
                if (r == c) siso += Jm23 * mu;
                S[3 * r + c] = wv * svol + s2 * siso;
            }
        double psip = tension ? U + psibar : psibar;
        double psim = tension ? 0.0 : U;
        out_psi[i] = s2 * psip + psim;
        out_psip[i] = psip;
    }
    return n_bad;
}

/* Finite-strain J2 radial return on the plastic metric Cp (in place, with
 * epbar).  reference.py:151-208, fast.py:335-423.  Returns n_bad; writes the
 * lowest non-SPD particle index (or -1) to *first_bad.  As in the reference
 * numpy path, a non-SPD update aborts before any state is committed. */
i64 orc_j2_batch(i64 n, const double *F, double *Cp, double *epbar, double mu, double kappa,
                 double sigma_y0, double H_hard, double *out_S, double *out_psi, double *out_dwp,
                 i64 *first_bad) {
    const double sq23 = sqrt(2.0 / 3.0);
    i64 n_bad = 0;
    i64 fb = -1;
    /* pass 1: detect a non-SPD update anywhere (reference aborts before commit) */
    double *Cp_new = (double *)malloc(sizeof(double) * 9 * (size_t)(n > 0 ? n : 1));
    unsigned char *plastic = (unsigned char *)calloc((size_t)(n > 0 ? n : 1), 1);
    unsigned char *bad = (unsigned char *)calloc((size_t)(n > 0 ? n : 1), 1);
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) {
        const double *Fi = F + 9 * i;
        double J = det3(Fi);
        if (J <= J_MIN) continue;
        double C[9], Cpi[9], Ce[9], Mdev[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                C[3 * r + c] = Fi[r] * Fi[c] + Fi[3 + r] * Fi[3 + c] + Fi[6 + r] * Fi[6 + c];
        inv3(Cp + 9 * i, Cpi);
        mm3(C, Cpi, Ce);
        double fac = pow(J, -2.0 / 3.0);
        double tr3 = fac * (Ce[0] + Ce[4] + Ce[8]) / 3.0;
        double frob = 0.0;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double m = mu * (fac * Ce[3 * r + c] - (r == c ? tr3 : 0.0));
                Mdev[3 * r + c] = m; frob += m * m;
            }
        double sigeq = sqrt(1.5 * frob);
        double sy = sigma_y0 + H_hard * epbar[i];
        if (sigeq - sy > 0.0) {
            double dg = (sigeq - sy) / (3.0 * mu + H_hard * sq23);
            double N[9], NC[9];
            for (int q = 0; q < 9; ++q) N[q] = (1.5 / sigeq) * Mdev[q];
            mm3(N, Cp + 9 * i, NC);
            double *cn = Cp_new + 9 * i;
            for (int q = 0; q < 9; ++q) cn[q] = Cp[9 * i + q] + 2.0 * dg * NC[q];
            for (int r = 0; r < 3; ++r)
                for (int c = r + 1; c < 3; ++c) {
                    double m = 0.5 * (cn[3 * r + c] + cn[3 * c + r]);
                    cn[3 * r + c] = cn[3 * c + r] = m;
                }
            plastic[i] = 1;
            if (det3(cn) <= 0.0) bad[i] = 1;
        }
    }
    for (i64 i = 0; i < n; ++i) if (bad[i]) { fb = i; break; }
    if (fb >= 0) {
        for (i64 i = 0; i < n; ++i) if (det3(F + 9 * i) <= J_MIN) n_bad += 1;
        free(Cp_new); free(plastic); free(bad);
        *first_bad = fb;
        return n_bad;
    }
#pragma omp parallel for schedule(static) reduction(+ : n_bad)
    for (i64 i = 0; i < n; ++i) {
        const double *Fi = F + 9 * i;
        double *S = out_S + 9 * i;
        double J = det3(Fi);
        if (J <= J_MIN) {
            for (int q = 0; q < 9; ++q) S[q] = 0.0;
            out_psi[i] = 0.0; out_dwp[i] = 0.0;
            n_bad += 1;
            continue;
        }
        double C[9], Cpi[9], Ce[9], Mdev[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                C[3 * r + c] = Fi[r] * Fi[c] + Fi[3 + r] * Fi[3 + c] + Fi[6 + r] * Fi[6 + c];
        inv3(Cp + 9 * i, Cpi);
        mm3(C, Cpi, Ce);
        double fac = pow(J, -2.0 / 3.0);
        double tr3 = fac * (Ce[0] + Ce[4] + Ce[8]) / 3.0;
        double frob = 0.0;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double m = mu * (fac * Ce[3 * r + c] - (r == c ? tr3 : 0.0));
                Mdev[3 * r + c] = m; frob += m * m;
            }
        double sigeq = sqrt(1.5 * frob);
        double sy = sigma_y0 + H_hard * epbar[i];
        double dwp = 0.0;
        if (plastic[i]) {
            double dg = (sigeq - sy) / (3.0 * mu + H_hard * sq23);
            double scale = 1.0 - 3.0 * mu * dg / sigeq;
            double *cn = Cp_new + 9 * i;
            double proj = pow(det3(cn), -1.0 / 3.0);
            for (int q = 0; q < 9; ++q) { Cp[9 * i + q] = cn[q] * proj; Mdev[q] *= scale; }
            double deb = sq23 * dg;
            dwp = (sy + 0.5 * H_hard * deb) * deb;
            epbar[i] += deb;
            inv3(Cp + 9 * i, Cpi);
            mm3(C, Cpi, Ce);
        }
        double Cei[9], Ci[9], T[9], Sd[9];
        inv3(Ce, Cei);
        inv3(C, Ci);
        mm3(Cei, Mdev, T);
        mm3(T, Cei, Sd);
        double vol = 0.5 * kappa * (J * J - 1.0);
        for (int q = 0; q < 9; ++q) S[q] = Sd[q] / J + vol * Ci[q];
        for (int r = 0; r < 3; ++r)
            for (int c = r + 1; c < 3; ++c) {
                double m = 0.5 * (S[3 * r + c] + S[3 * c + r]);
                S[3 * r + c] = S[3 * c + r] = m;
            }
        double trbar = fac * (Ce[0] + Ce[4] + Ce[8]);
        out_psi[i] = 0.25 * kappa * (J * J - 1.0 - 2.0 * log(J)) + 0.5 * mu * (trbar - 3.0);
        out_dwp[i] = dwp;
    }
    free(Cp_new); free(plastic); free(bad);
    *first_bad = -1;
    return n_bad;
}

/* Penalty contact over precomputed cross-body pairs (sequential; equal and
 * opposite forces).  reference.py:211-244. */
i64 orc_contact_pair_accumulate(const double *xa, const double *va, const double *ma,
                                const double *xb, const double *vb, const double *mb,
                                i64 npairs, const i64 *pairs, double dpc, double k_n,
                                double c_n, double kfric, double *out_aa, double *out_ab) {
    i64 n_warn = 0;
    for (i64 k = 0; k < npairs; ++k) {
        i64 i = pairs[2 * k], j = pairs[2 * k + 1];
        double d[3], nv[3], dv[3];
        for (int a = 0; a < 3; ++a) d[a] = xa[3 * i + a] - xb[3 * j + a];
        double dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        if (dist >= dpc) continue;
        if (dist < 1e-12) { nv[0] = 1.0; nv[1] = 0.0; nv[2] = 0.0; dist = 1e-12; n_warn += 1; }
        else for (int a = 0; a < 3; ++a) nv[a] = d[a] / dist;
        double overlap = dpc - dist;
        for (int a = 0; a < 3; ++a) dv[a] = va[3 * i + a] - vb[3 * j + a];
        double vn = dv[0] * nv[0] + dv[1] * nv[1] + dv[2] * nv[2];
        double fn = k_n * overlap - c_n * vn;
        if (fn < 0.0) fn = 0.0;
        double f[3];
        for (int a = 0; a < 3; ++a) f[a] = fn * nv[a];
        if (kfric > 0.0) {
            double t[3];
            for (int a = 0; a < 3; ++a) t[a] = dv[a] - vn * nv[a];
            double vt = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
            if (vt > 1e-14)
                for (int a = 0; a < 3; ++a) f[a] -= kfric * fn * t[a] / vt;
        }
        for (int a = 0; a < 3; ++a) {
            out_aa[3 * i + a] += f[a] / ma[i];
            out_ab[3 * j + a] -= f[a] / mb[j];
        }
    }
    return n_warn;
}

/* ---- reference-configuration neighbour search (kernel_geom.py:65-97) --
 * Exact inclusion tests, evaluated in the order numpy 2.3 evaluates them:
 *   radial:   fl(fl(dx*dx + dz*dz) + dy*dy) < (2h)^2      (einsum order)
 *   nbsrange: |dx|<=win && |dy|<=win && |dz|<=win
 * The cKDTree prefilter in the reference only removes far pairs, so a cell
 * list with cells >= the cutoff finds the same set.  Output: per-row counts
 * (count pass) or the CSR column list in ascending j (fill pass). */
typedef struct {
    i64 n;
    const double *X;
    int nbs;
    double cut2, win;
    double lo[3], cell;
    i64 dims[3];
    i64 *cell_start; /* ncell + 1 */
    i64 *order;      /* particles sorted by cell, ascending index within */
} orc_grid;

static int pair_keep(const orc_grid *g, i64 a, i64 b) {
    const double *X = g->X;
    double dx = X[3 * a] - X[3 * b], dy = X[3 * a + 1] - X[3 * b + 1], dz = X[3 * a + 2] - X[3 * b + 2];
    if (g->nbs) return fabs(dx) <= g->win && fabs(dy) <= g->win && fabs(dz) <= g->win;
    double s = dx * dx + dz * dz;
    s = s + dy * dy;
    return s < g->cut2;
}

static int cmp_i64(const void *a, const void *b) {
    i64 x = *(const i64 *)a, y = *(const i64 *)b;
    return (x > y) - (x < y);
}

/* counts[i] = number of kept partners of i; if cols != NULL also fills the
 * CSR (cols at indptr[i]..) in ascending partner order. */
int orc_build_pairs(i64 n, const double *X, int nbs, double h, double win, i64 *counts,
                    const i64 *indptr, i64 *cols) {
    orc_grid g;
    g.n = n; g.X = X; g.nbs = nbs;
    g.cut2 = (2.0 * h) * (2.0 * h);
    g.win = win;
    double reach = nbs ? win : 2.0 * h;
    g.cell = reach * (1.0 + 1e-6);
    double hi[3];
    for (int a = 0; a < 3; ++a) { g.lo[a] = INFINITY; hi[a] = -INFINITY; }
    for (i64 i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            if (X[3 * i + a] < g.lo[a]) g.lo[a] = X[3 * i + a];
            if (X[3 * i + a] > hi[a]) hi[a] = X[3 * i + a];
        }
    i64 ncell = 1;
    for (int a = 0; a < 3; ++a) {
        g.dims[a] = (i64)floor((hi[a] - g.lo[a]) / g.cell) + 1;
        ncell *= g.dims[a];
    }
    i64 *cid = (i64 *)malloc(sizeof(i64) * (size_t)n);
    g.cell_start = (i64 *)calloc((size_t)ncell + 1, sizeof(i64));
    g.order = (i64 *)malloc(sizeof(i64) * (size_t)n);
    for (i64 i = 0; i < n; ++i) {
        i64 c[3];
        for (int a = 0; a < 3; ++a) {
            c[a] = (i64)floor((X[3 * i + a] - g.lo[a]) / g.cell);
            if (c[a] >= g.dims[a]) c[a] = g.dims[a] - 1;
        }
        cid[i] = (c[0] * g.dims[1] + c[1]) * g.dims[2] + c[2];
        g.cell_start[cid[i] + 1] += 1;
    }
    for (i64 c = 0; c < ncell; ++c) g.cell_start[c + 1] += g.cell_start[c];
    i64 *fillp = (i64 *)malloc(sizeof(i64) * (size_t)ncell);
    memcpy(fillp, g.cell_start, sizeof(i64) * (size_t)ncell);
    for (i64 i = 0; i < n; ++i) g.order[fillp[cid[i]]++] = i;
    free(fillp);
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 i = 0; i < n; ++i) {
        i64 c0 = cid[i] / (g.dims[1] * g.dims[2]);
        i64 c1 = (cid[i] / g.dims[2]) % g.dims[1];
        i64 c2 = cid[i] % g.dims[2];
        i64 cnt = 0;
        i64 *out = cols ? cols + indptr[i] : NULL;
        for (i64 a = c0 - 1; a <= c0 + 1; ++a) {
            if (a < 0 || a >= g.dims[0]) continue;
            for (i64 b = c1 - 1; b <= c1 + 1; ++b) {
                if (b < 0 || b >= g.dims[1]) continue;
                for (i64 c = c2 - 1; c <= c2 + 1; ++c) {
                    if (c < 0 || c >= g.dims[2]) continue;
                    i64 cc = (a * g.dims[1] + b) * g.dims[2] + c;
                    for (i64 p = g.cell_start[cc]; p < g.cell_start[cc + 1]; ++p) {
                        i64 j = g.order[p];
                        if (j == i) continue;
                        /* the reference tests X[min]-X[max] (query_pairs gives i<j) */
                        int keep = i < j ? pair_keep(&g, i, j) : pair_keep(&g, j, i);
                        if (keep) {
                            if (out) out[cnt] = j;
                            ++cnt;
                        }
                    }
                }
            }
        }
        if (out) qsort(out, (size_t)cnt, sizeof(i64), cmp_i64);
        counts[i] = cnt;
    }
    free(cid); free(g.cell_start); free(g.order);
    return 0;
}

/* First-order correction moment matrices and inverses.
 * kernel_geom.py:176-205: A_i = sum_j V0_j gb_ij (x) (X_j - X_i) in CSR order;
 * 2D: y row/col -> identity; L_i = inv(A_i) when finite and cond_2 < 1e8, else
 * I (counted).  numpy uses the SVD for cond_2; see the note in the body. */
i64 orc_correction(i64 n, const i64 *indptr, const i64 *indices, const double *X,
                   const double *V0, const double *grad_base, int dim, double *A_out, double *L) {
    i64 fallbacks = 0;
#pragma omp parallel for schedule(static) reduction(+ : fallbacks)
    for (i64 i = 0; i < n; ++i) {
        double A[9] = {0};
        for (i64 k = indptr[i]; k < indptr[i + 1]; ++k) {
            i64 j = indices[k];
            double d[3];
            for (int a = 0; a < 3; ++a) d[a] = X[3 * j + a] - X[3 * i + a];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) A[3 * r + c] += V0[j] * grad_base[3 * k + r] * d[c];
        }
        if (dim == 2) {
            for (int c = 0; c < 3; ++c) { A[3 + c] = 0.0; A[3 * c + 1] = 0.0; }
            A[4] = 1.0;
        }
        if (A_out) memcpy(A_out + 9 * i, A, sizeof A);
        int finite = 1;
        for (int q = 0; q < 9; ++q) if (!isfinite(A[q])) finite = 0;
        /* cond_2 = sigma_max(A) * sigma_max(A^-1): both largest eigenvalues
         * of a Gram matrix, which Jacobi resolves to full relative accuracy */
        double cond = INFINITY;
        double Ai[9];
        if (finite && det3(A) != 0.0) {
            inv3(A, Ai);
            double G[9], Gi[9], w[3], Q[9];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) {
                    G[3 * r + c] = A[r] * A[c] + A[3 + r] * A[3 + c] + A[6 + r] * A[6 + c];
                    Gi[3 * r + c] = Ai[r] * Ai[c] + Ai[3 + r] * Ai[3 + c] + Ai[6 + r] * Ai[6 + c];
                }
            orc_eig3_jacobi(G, w, Q);
            double smax = sqrt(w[0]);
            orc_eig3_jacobi(Gi, w, Q);
            cond = smax * sqrt(w[0]);
            if (!isfinite(cond)) cond = INFINITY;
        }
        double *Li = L + 9 * i;
        if (finite && isfinite(cond) && cond < 1.0e8) {
            memcpy(Li, Ai, sizeof Ai);
        } else {
            for (int q = 0; q < 9; ++q) Li[q] = (q % 4 == 0) ? 1.0 : 0.0;
            fallbacks += 1;
        }
    }
    return fallbacks;
}
