// plugin.cu -- ABI plumbing and the backend-plugin kernels.
//
// These mirror the 8 kernels of the reference backend plugin on device
// pointers (reference backends/reference.py:18-244, backends/fast.py:111-469):
// the per-pair arrays (grad0, grad0r, r0, r0norm) are the reference
// Adjacency's, FP64, and each thread owns one particle and sums its CSR row
// sequentially -- the same accumulation order as np.add.at.  They serve the
// kernel-level drop-in (paper_2602_15149_b200/backend.py).  The throughput
// path is the fused pass A / pass B in step.cu, which does not store per-pair
// arrays at all.
#include <cstdarg>
#include <cstdio>

#include "tl_common.cuh"

static thread_local char g_err[512] = "";

void tl_set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int tl_check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        tl_set_error("%s launch failed: %s", what, cudaGetErrorString(e));
        return TL_ERR_CUDA;
    }
    return TL_OK;
}

bool tl_pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("TLSPH_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

extern "C" int tl_abi_version(void) { return TL_ABI_VERSION; }
extern "C" int64_t tl_struct_size(int which) {
    switch (which) {
        case 0: return (int64_t)sizeof(tl_body);
        case 1: return (int64_t)sizeof(tl_clock);
        case 2: return (int64_t)sizeof(tl_bc);
        case 3: return (int64_t)sizeof(tl_prog);
        case 4: return (int64_t)sizeof(tl_notch);
        case 5: return (int64_t)sizeof(tl_nb_params);
        case 6: return (int64_t)sizeof(tl_dtinfo);
        case 7: return (int64_t)sizeof(tl_contact_side);
        default: return -1;
    }
}
extern "C" const char* tl_last_error(void) { return g_err; }
extern "C" int tl_device_sync(void) {
    TL_TRY_CUDA(cudaDeviceSynchronize());
    return TL_OK;
}

using tl::det3;
using tl::inv3;
using tl::mm3;

namespace {

constexpr int kThreads = 256;

__global__ void k_deformation_gradient(int64_t n, const int64_t* __restrict__ indptr,
                                       const int64_t* __restrict__ indices,
                                       const double* __restrict__ grad0,
                                       const double* __restrict__ u, const double* __restrict__ V0,
                                       const double* __restrict__ s, double s_l, int gated,
                                       double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double f[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    if (!(gated && s[i] <= s_l)) {
        const double ui0 = u[3 * i], ui1 = u[3 * i + 1], ui2 = u[3 * i + 2];
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
            const int64_t j = indices[k];
            const double vj = V0[j];
            const double d[3] = {__dmul_rn(vj, __dsub_rn(u[3 * j], ui0)),
                                 __dmul_rn(vj, __dsub_rn(u[3 * j + 1], ui1)),
                                 __dmul_rn(vj, __dsub_rn(u[3 * j + 2], ui2))};
            const double g[3] = {grad0[3 * k], grad0[3 * k + 1], grad0[3 * k + 2]};
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) f[3 * a + b] = __dadd_rn(f[3 * a + b], __dmul_rn(d[a], g[b]));
        }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) out[9 * i + q] = f[q];
}

__global__ void k_sph_laplacian(int64_t n, const int64_t* __restrict__ indptr,
                                const int64_t* __restrict__ indices,
                                const double* __restrict__ grad0, const double* __restrict__ r0,
                                const double* __restrict__ r0norm, const double* __restrict__ V0,
                                const double* __restrict__ f, double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    const double fi = f[i];
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
        const int64_t j = indices[k];
        double rdg = r0[3 * k] * grad0[3 * k] + r0[3 * k + 1] * grad0[3 * k + 1] +
                     r0[3 * k + 2] * grad0[3 * k + 2];
        acc += 2.0 * (fi - f[j]) * V0[j] * rdg / (r0norm[k] * r0norm[k]);
    }
    out[i] = acc;
}

__global__ void k_sph_gradient(int64_t n, const int64_t* __restrict__ indptr,
                               const int64_t* __restrict__ indices,
                               const double* __restrict__ grad0, const double* __restrict__ V0,
                               const double* __restrict__ f, double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double g0 = 0, g1 = 0, g2 = 0;
    const double fi = f[i];
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
        const int64_t j = indices[k];
        const double c = __dmul_rn(V0[j], __dsub_rn(f[j], fi));
        g0 = __dadd_rn(g0, __dmul_rn(c, grad0[3 * k]));
        g1 = __dadd_rn(g1, __dmul_rn(c, grad0[3 * k + 1]));
        g2 = __dadd_rn(g2, __dmul_rn(c, grad0[3 * k + 2]));
    }
    out[3 * i] = g0;
    out[3 * i + 1] = g1;
    out[3 * i + 2] = g2;
}

__global__ void k_momentum(int64_t n, const int64_t* __restrict__ indptr,
                           const int64_t* __restrict__ indices, const double* __restrict__ grad0,
                           const double* __restrict__ grad0r, const double* __restrict__ r0,
                           const double* __restrict__ r0norm, const double* __restrict__ P,
                           const double* __restrict__ m0, double rho0,
                           const double* __restrict__ v, double h, double c0, double beta1,
                           double beta2, const double* __restrict__ F, double* __restrict__ out,
                           int64_t* n_bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int bad = 0;
    if (i < n) {
        const bool visc = beta1 != 0.0 || beta2 != 0.0;
        const double inv_rho2 = 1.0 / (rho0 * rho0);
        const double eps_h2 = 0.001 * h * h;
        double Av[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (visc) {
            double Fi[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) Fi[q] = F[9 * i + q];
            const double d = det3(Fi);
            if (d > TL_J_MIN) {
                inv3(Fi, Av);
#pragma unroll
                for (int q = 0; q < 9; ++q) Av[q] *= d;
            } else {
                bad = 1;
            }
        }
        double Pi[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) Pi[q] = P[9 * i + q];
        const double vi0 = v[3 * i], vi1 = v[3 * i + 1], vi2 = v[3 * i + 2];
        double a0 = 0, a1 = 0, a2 = 0;
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
            const int64_t j = indices[k];
            const double g[3] = {grad0[3 * k], grad0[3 * k + 1], grad0[3 * k + 2]};
            const double q[3] = {grad0r[3 * k], grad0r[3 * k + 1], grad0r[3 * k + 2]};
            const double* Pj = P + 9 * j;
            double fp[3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
                fp[a] = ((Pi[3 * a] * g[0] + Pi[3 * a + 1] * g[1] + Pi[3 * a + 2] * g[2]) -
                         (Pj[3 * a] * q[0] + Pj[3 * a + 1] * q[1] + Pj[3 * a + 2] * q[2])) *
                        inv_rho2;
            if (visc) {
                const double G = h *
                                 ((vi0 - v[3 * j]) * r0[3 * k] + (vi1 - v[3 * j + 1]) * r0[3 * k + 1] +
                                  (vi2 - v[3 * j + 2]) * r0[3 * k + 2]) /
                                 (r0norm[k] * r0norm[k] + eps_h2);
                const double pi = (beta2 * G * G - beta1 * c0 * G) / rho0;
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    fp[a] -= pi * (Av[3 * a] * g[0] + Av[3 * a + 1] * g[1] + Av[3 * a + 2] * g[2]);
            }
            const double mj = m0[j];
            a0 += mj * fp[0];
            a1 += mj * fp[1];
            a2 += mj * fp[2];
        }
        out[3 * i] = a0;
        out[3 * i + 1] = a1;
        out[3 * i + 2] = a2;
    }
    int nb = tl::warp_sum_int(bad);
    if ((threadIdx.x & 31) == 0 && nb) atomicAdd((unsigned long long*)n_bad, (unsigned long long)nb);
}

__global__ void k_svk(int64_t n, const double* __restrict__ F, double lam, double mu,
                      const double* __restrict__ s, int fracture, double* __restrict__ S,
                      double* __restrict__ psi, double* __restrict__ psip, int64_t* n_noconv) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int nc = 0;
    if (i < n) {
        const double* Fi = F + 9 * i;
        double E[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                E[3 * r + c] = 0.5 * ((Fi[r] * Fi[c] + Fi[3 + r] * Fi[3 + c] + Fi[6 + r] * Fi[6 + c]) -
                                      (r == c ? 1.0 : 0.0));
        E[1] = E[3] = 0.5 * (E[1] + E[3]);
        E[2] = E[6] = 0.5 * (E[2] + E[6]);
        E[5] = E[7] = 0.5 * (E[5] + E[7]);
        const double trE = E[0] + E[4] + E[8];
        double* Si = S + 9 * i;
        if (!fracture) {
            double frob = 0.0;
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                Si[q] = 2.0 * mu * E[q] + ((q % 4 == 0) ? lam * trE : 0.0);
                frob += E[q] * E[q];
            }
            psi[i] = 0.5 * lam * trE * trE + mu * frob;
            psip[i] = 0.0;
        } else {
            double w[3], Q[9];
            if (tl::eig3_jacobi(E, w, Q, 1e-30) >= 64) nc = 1;
            const double trp = trE > 0.0 ? trE : 0.0, trm = trE < 0.0 ? trE : 0.0;
            double pp = 0.5 * lam * trp * trp, pm = 0.5 * lam * trm * trm;
            const double s2 = s[i] * s[i];
            double lp[3], lm[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                lp[k] = w[k] > 0.0 ? w[k] : 0.0;
                lm[k] = w[k] < 0.0 ? w[k] : 0.0;
            }
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double ep = 0.0, em = 0.0;
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        ep += Q[3 * r + k] * lp[k] * Q[3 * c + k];
                        em += Q[3 * r + k] * lm[k] * Q[3 * c + k];
                    }
                    double sp = 2.0 * mu * ep, sm = 2.0 * mu * em;
                    if (r == c) {
                        sp += lam * trp;
                        sm += lam * trm;
                    }
                    Si[3 * r + c] = s2 * sp + sm;
                }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                pp += mu * lp[k] * lp[k];
                pm += mu * lm[k] * lm[k];
            }
            psi[i] = s2 * pp + pm;
            psip[i] = pp;
        }
    }
    int t = tl::warp_sum_int(nc);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd((unsigned long long*)n_noconv, (unsigned long long)t);
}

__global__ void k_nh(int64_t n, const double* __restrict__ F, double kappa, double mu,
                     const double* __restrict__ s, int fracture, double* __restrict__ S,
                     double* __restrict__ psi, double* __restrict__ psip, int64_t* n_bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int bad = 0;
    if (i < n) {
        const double* Fi = F + 9 * i;
        double* Si = S + 9 * i;
        const double J = det3(Fi);
        if (J <= TL_J_MIN) {
#pragma unroll
            for (int q = 0; q < 9; ++q) Si[q] = 0.0;
            psi[i] = 0.0;
            psip[i] = 0.0;
            bad = 1;
        } else {
            double b[9], bi[9];
            tl::mmT3(Fi, Fi, b);
            inv3(b, bi);
            const double trb = b[0] + b[4] + b[8];
            const double Jm23 = pow(J, -2.0 / 3.0);
            const double U = 0.5 * kappa * (0.5 * (J * J - 1.0) - log(J));
            const double pbar = 0.5 * mu * (Jm23 * trb - 3.0);
            const double s2 = fracture ? s[i] * s[i] : 1.0;
            const bool tension = J >= 1.0;
            const double wv = tension ? s2 : 1.0;
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                const double svol = 0.5 * kappa * (J * J - 1.0) * bi[q];
                double siso = Jm23 * mu * (-(trb / 3.0) * bi[q]);
                if (q % 4 == 0) siso += Jm23 * mu;
                Si[q] = wv * svol + s2 * siso;
            }
            const double pp = tension ? U + pbar : pbar;
            const double pm = tension ? 0.0 : U;
            psi[i] = s2 * pp + pm;
            psip[i] = pp;
        }
    }
    int t = tl::warp_sum_int(bad);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd((unsigned long long*)n_bad, (unsigned long long)t);
}

// J2 trial + return.  Phase 0 flags plastic lanes whose Cp update would be
// non-SPD (reference aborts before committing any state, reference.py:182-187);
// phase 1 commits.
__device__ void j2_trial(const double* Fi, const double* Cpi, double epb, double mu,
                         double sigma_y0, double H_hard, double* C, double* Ce, double* Mdev,
                         double& J, double& fac, double& sigeq, double& sy) {
    J = det3(Fi);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            C[3 * r + c] = Fi[r] * Fi[c] + Fi[3 + r] * Fi[3 + c] + Fi[6 + r] * Fi[6 + c];
    double Cpinv[9];
    inv3(Cpi, Cpinv);
    mm3(C, Cpinv, Ce);
    fac = pow(J, -2.0 / 3.0);
    const double tr3 = fac * (Ce[0] + Ce[4] + Ce[8]) / 3.0;
    double frob = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        const double m = mu * (fac * Ce[q] - ((q % 4 == 0) ? tr3 : 0.0));
        Mdev[q] = m;
        frob += m * m;
    }
    sigeq = sqrt(1.5 * frob);
    sy = sigma_y0 + H_hard * epb;
}

__device__ void j2_flow(const double* Cpi, const double* Mdev, double dg, double sigeq,
                        double* Cn) {
    double N[9], NC[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) N[q] = (1.5 / sigeq) * Mdev[q];
    mm3(N, Cpi, NC);
#pragma unroll
    for (int q = 0; q < 9; ++q) Cn[q] = Cpi[q] + 2.0 * dg * NC[q];
    Cn[1] = Cn[3] = 0.5 * (Cn[1] + Cn[3]);
    Cn[2] = Cn[6] = 0.5 * (Cn[2] + Cn[6]);
    Cn[5] = Cn[7] = 0.5 * (Cn[5] + Cn[7]);
}

__global__ void k_j2_check(int64_t n, const double* __restrict__ F, const double* __restrict__ Cp,
                           const double* __restrict__ epbar, double mu, double sigma_y0,
                           double H_hard, int64_t* counters) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* Fi = F + 9 * i;
    if (det3(Fi) <= TL_J_MIN) return;
    double C[9], Ce[9], Mdev[9], J, fac, sigeq, sy;
    j2_trial(Fi, Cp + 9 * i, epbar[i], mu, sigma_y0, H_hard, C, Ce, Mdev, J, fac, sigeq, sy);
    if (sigeq - sy > 0.0) {
        const double dg = (sigeq - sy) / (3.0 * mu + H_hard * sqrt(2.0 / 3.0));
        double Cn[9];
        j2_flow(Cp + 9 * i, Mdev, dg, sigeq, Cn);
        if (det3(Cn) <= 0.0) atomicMin((long long*)&counters[1], (long long)i);
    }
}

__global__ void k_j2_commit(int64_t n, const double* __restrict__ F, double* __restrict__ Cp,
                            double* __restrict__ epbar, double mu, double kappa, double sigma_y0,
                            double H_hard, double* __restrict__ S, double* __restrict__ psi,
                            double* __restrict__ dwp, int64_t* counters) {
    if (counters[1] != INT64_MAX) return;  // non-SPD somewhere: nothing committed
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int bad = 0;
    if (i < n) {
        const double* Fi = F + 9 * i;
        double* Si = S + 9 * i;
        if (det3(Fi) <= TL_J_MIN) {
#pragma unroll
            for (int q = 0; q < 9; ++q) Si[q] = 0.0;
            psi[i] = 0.0;
            dwp[i] = 0.0;
            bad = 1;
        } else {
            double* Cpi = Cp + 9 * i;
            double C[9], Ce[9], Mdev[9], J, fac, sigeq, sy;
            j2_trial(Fi, Cpi, epbar[i], mu, sigma_y0, H_hard, C, Ce, Mdev, J, fac, sigeq, sy);
            double w = 0.0;
            if (sigeq - sy > 0.0) {
                const double sq23 = sqrt(2.0 / 3.0);
                const double dg = (sigeq - sy) / (3.0 * mu + H_hard * sq23);
                const double scale = 1.0 - 3.0 * mu * dg / sigeq;
                double Cn[9];
                j2_flow(Cpi, Mdev, dg, sigeq, Cn);
                const double proj = pow(det3(Cn), -1.0 / 3.0);
#pragma unroll
                for (int q = 0; q < 9; ++q) {
                    Cpi[q] = Cn[q] * proj;
                    Mdev[q] *= scale;
                }
                const double deb = sq23 * dg;
                w = (sy + 0.5 * H_hard * deb) * deb;
                epbar[i] += deb;
                double Cpinv[9];
                inv3(Cpi, Cpinv);
                mm3(C, Cpinv, Ce);
            }
            double Cei[9], Ci[9], T[9], Sd[9];
            inv3(Ce, Cei);
            inv3(C, Ci);
            mm3(Cei, Mdev, T);
            mm3(T, Cei, Sd);
            const double vol = 0.5 * kappa * (J * J - 1.0);
#pragma unroll
            for (int q = 0; q < 9; ++q) Si[q] = Sd[q] / J + vol * Ci[q];
            Si[1] = Si[3] = 0.5 * (Si[1] + Si[3]);
            Si[2] = Si[6] = 0.5 * (Si[2] + Si[6]);
            Si[5] = Si[7] = 0.5 * (Si[5] + Si[7]);
            const double trbar = fac * (Ce[0] + Ce[4] + Ce[8]);
            psi[i] = 0.25 * kappa * (J * J - 1.0 - 2.0 * log(J)) + 0.5 * mu * (trbar - 3.0);
            dwp[i] = w;
        }
    }
    int t = tl::warp_sum_int(bad);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd((unsigned long long*)&counters[0], (unsigned long long)t);
}

__global__ void k_contact_pairs(const double* xa, const double* va, const double* xb,
                                const double* vb, int64_t np, const int64_t* pairs, double dpc,
                                double k_n, double c_n, double kfric, double* force,
                                int64_t* n_warn) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= np) return;
    const int64_t i = pairs[2 * k], j = pairs[2 * k + 1];
    double d[3], nv[3], dv[3];
    for (int a = 0; a < 3; ++a) d[a] = xa[3 * i + a] - xb[3 * j + a];
    double dist = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    force[3 * k] = force[3 * k + 1] = force[3 * k + 2] = 0.0;
    if (dist >= dpc) {
        force[3 * k] = nan("");  // marks "no contact" (pair skipped)
        return;
    }
    if (dist < 1e-12) {
        nv[0] = 1.0; nv[1] = 0.0; nv[2] = 0.0;
        dist = 1e-12;
        atomicAdd((unsigned long long*)n_warn, 1ull);
    } else {
        for (int a = 0; a < 3; ++a) nv[a] = d[a] / dist;
    }
    const double overlap = dpc - dist;
    for (int a = 0; a < 3; ++a) dv[a] = va[3 * i + a] - vb[3 * j + a];
    const double vn = dv[0] * nv[0] + dv[1] * nv[1] + dv[2] * nv[2];
    double fn = k_n * overlap - c_n * vn;
    if (fn < 0.0) fn = 0.0;
    double f[3];
    for (int a = 0; a < 3; ++a) f[a] = fn * nv[a];
    if (kfric > 0.0) {
        double t[3];
        for (int a = 0; a < 3; ++a) t[a] = dv[a] - vn * nv[a];
        const double vt = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
        if (vt > 1e-14)
            for (int a = 0; a < 3; ++a) f[a] -= kfric * fn * t[a] / vt;
    }
    for (int a = 0; a < 3; ++a) force[3 * k + a] = f[a];
}

// sequential accumulation in pair order (the reference's loop order)
__global__ void k_contact_accumulate(const double* ma, const double* mb, int64_t np,
                                     const int64_t* pairs, const double* force, double* aa,
                                     double* ab) {
    for (int64_t k = 0; k < np; ++k) {
        if (isnan(force[3 * k])) continue;
        const int64_t i = pairs[2 * k], j = pairs[2 * k + 1];
        for (int a = 0; a < 3; ++a) {
            aa[3 * i + a] += force[3 * k + a] / ma[i];
            ab[3 * j + a] -= force[3 * k + a] / mb[j];
        }
    }
}

__global__ void k_eig(int64_t n, const double* A, double* w, double* Q, int32_t* sweeps) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    sweeps[i] = tl::eig3_jacobi(A + 9 * i, w + 3 * i, Q + 9 * i, 1e-30);
}

}  // namespace

#define LAUNCH(kern, n, st, ...)                                                   \
    do {                                                                           \
        if ((n) > 0)                                                               \
            kern<<<tl_blocks((n), kThreads), kThreads, 0, (cudaStream_t)(st)>>>(__VA_ARGS__); \
        return tl_check_launch(#kern);                                             \
    } while (0)

extern "C" int tl_deformation_gradient(tl_stream_t st, int64_t n, const int64_t* indptr,
                                       const int64_t* indices, const double* grad0,
                                       const double* u, const double* V0, const double* s,
                                       double s_l, int gated, double* out) {
    LAUNCH(k_deformation_gradient, n, st, n, indptr, indices, grad0, u, V0, s, s_l, gated, out);
}

extern "C" int tl_sph_laplacian(tl_stream_t st, int64_t n, const int64_t* indptr,
                                const int64_t* indices, const double* grad0, const double* r0,
                                const double* r0norm, const double* V0, const double* f,
                                double* out) {
    LAUNCH(k_sph_laplacian, n, st, n, indptr, indices, grad0, r0, r0norm, V0, f, out);
}

extern "C" int tl_sph_gradient(tl_stream_t st, int64_t n, const int64_t* indptr,
                               const int64_t* indices, const double* grad0, const double* V0,
                               const double* f, double* out) {
    LAUNCH(k_sph_gradient, n, st, n, indptr, indices, grad0, V0, f, out);
}

extern "C" int tl_momentum(tl_stream_t st, int64_t n, const int64_t* indptr,
                           const int64_t* indices, const double* grad0, const double* grad0r,
                           const double* r0, const double* r0norm, const double* P,
                           const double* m0, double rho0, const double* v, double h, double c0,
                           double beta1, double beta2, const double* F, double* out,
                           int64_t* n_bad) {
    LAUNCH(k_momentum, n, st, n, indptr, indices, grad0, grad0r, r0, r0norm, P, m0, rho0, v, h,
           c0, beta1, beta2, F, out, n_bad);
}

extern "C" int tl_svk_batch(tl_stream_t st, int64_t n, const double* F, double lam, double mu,
                            const double* s, int fracture, double* out_S, double* out_psi,
                            double* out_psip, int64_t* n_noconv) {
    LAUNCH(k_svk, n, st, n, F, lam, mu, s, fracture, out_S, out_psi, out_psip, n_noconv);
}

extern "C" int tl_nh_batch(tl_stream_t st, int64_t n, const double* F, double kappa, double mu,
                           const double* s, int fracture, double* out_S, double* out_psi,
                           double* out_psip, int64_t* n_bad) {
    LAUNCH(k_nh, n, st, n, F, kappa, mu, s, fracture, out_S, out_psi, out_psip, n_bad);
}

extern "C" int tl_j2_batch(tl_stream_t st, int64_t n, const double* F, double* Cp, double* epbar,
                           double mu, double kappa, double sigma_y0, double H_hard, double* out_S,
                           double* out_psi, double* out_dwp, int64_t* counters, uint8_t*) {
    if (n <= 0) return TL_OK;
    cudaStream_t s = (cudaStream_t)st;
    k_j2_check<<<tl_blocks(n, kThreads), kThreads, 0, s>>>(n, F, Cp, epbar, mu, sigma_y0, H_hard,
                                                          counters);
    int rc = tl_check_launch("k_j2_check");
    if (rc) return rc;
    k_j2_commit<<<tl_blocks(n, kThreads), kThreads, 0, s>>>(n, F, Cp, epbar, mu, kappa, sigma_y0,
                                                           H_hard, out_S, out_psi, out_dwp,
                                                           counters);
    return tl_check_launch("k_j2_commit");
}

extern "C" int tl_contact_pair_accumulate(tl_stream_t st, const double* xa, const double* va,
                                          const double* ma, const double* xb, const double* vb,
                                          const double* mb, int64_t npairs, const int64_t* pairs,
                                          double dpc, double k_n, double c_n, double kfric,
                                          double* out_aa, double* out_ab, int64_t* n_warn,
                                          double* scratch) {
    if (npairs <= 0) return TL_OK;
    cudaStream_t s = (cudaStream_t)st;
    k_contact_pairs<<<tl_blocks(npairs, kThreads), kThreads, 0, s>>>(
        xa, va, xb, vb, npairs, pairs, dpc, k_n, c_n, kfric, scratch, n_warn);
    int rc = tl_check_launch("k_contact_pairs");
    if (rc) return rc;
    k_contact_accumulate<<<1, 1, 0, s>>>(ma, mb, npairs, pairs, scratch, out_aa, out_ab);
    return tl_check_launch("k_contact_accumulate");
}

extern "C" int tl_eig3_jacobi(tl_stream_t st, int64_t n, const double* A, double* w, double* Q,
                              int32_t* sweeps) {
    LAUNCH(k_eig, n, st, n, A, w, Q, sweeps);
}
