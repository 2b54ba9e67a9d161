// step.cu -- the fused, device-resident TLSPH step.
//
// Two gather passes per force evaluation replace the reference's per-step
// call chain (stepper.py:77-100 -> dynamics/constitutive/fracture ->
// backends.*):
//
//   pass A  (per particle i, neighbours j in CSR order)
//       D_i  = sum_j V0_j fac_ij (u_j - u_i) (x) r0_ij          F = I + D L_i^T
//       M_i  = sum_j 2 (s_i - s_j) V0_j fac_ij / r_ij^2 r0 r0^T  lap = L_i : M_i
//     then the constitutive model (SVK + spectral split | neo-Hookean | J2),
//     history H = max(psi+, H), s-ddot, and the two per-particle tensors the
//     momentum pass needs: PL_i = F S L_i and AL_i = det(F) F^-1 L_i.
//   pass B
//       a_i = (PL_i s1 + s2)/rho0^2 - AL_i s3  with
//       s1 = sum m_j fac r0,  s2 = sum m_j fac PL_j r0,
//       s3 = sum m_j fac pi_ij r0
//     then f0, force BCs, velocity BCs, the Verlet / symplectic update, the
//     phase-field advance and clamps, and the dt maxima.
//
// Identity used: the reference's corrected gradients are grad0_ij = L_i gb_ij
// and grad0r_ij = -L_j gb_ij with gb_ij = fac_ij r0_ij (kernel_geom.py:241-250),
// so every L is applied once per particle instead of per pair, and no per-pair
// array is stored -- only positions (FP64), L_i and the CSR.  Neighbour sums
// run sequentially in the reference's CSR order, one thread per particle;
// neighbour indices come from a lane-interleaved sliced-ELL copy of the CSR
// so every index load is one coalesced 128-byte line per warp.
//
// FP32 mode keeps reference-configuration differences in FP64 and carries
// H = F - I so strains do not cancel.
#include <cfloat>

#include "expr_vm.cuh"
#include "tl_common.cuh"

namespace {

using tl::det3;
using tl::inv3;
using tl::mm3;

constexpr int kThreads = 256;

__device__ __forceinline__ bool halted(const tl_body& b) {
    return b.clock != nullptr && *(volatile int32_t*)&b.clock->halted != 0;
}

// host-layout FP64 mirrors are written when the host asked for them on every
// step (write_out) or the device clock flags this step as ending on an output
// boundary, so run() never re-evaluates stress just to report it
__device__ __forceinline__ bool mirror_out(const tl_body& b) {
    return b.F_out != nullptr && (b.write_out || (b.clock != nullptr && b.clock->out_step));
}

// ---------------------------------------------------------------------------
// constitutive models on F = I + H (H-form)
// ---------------------------------------------------------------------------

// SVK with optional spectral split (reference.py:94-116, fast.py:224-284)
template <typename R>
__device__ __forceinline__ int svk_update(const R* H, R lam, R mu, R s, bool fracture, R jtol,
                                          R* S, R& psi, R& psip) {
    R E[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            E[3 * r + c] = R(0.5) * (H[3 * r + c] + H[3 * c + r] +
                                     (H[r] * H[c] + H[3 + r] * H[3 + c] + H[6 + r] * H[6 + c]));
    const R trE = E[0] + E[4] + E[8];
    if (!fracture) {
        R frob = R(0);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            S[q] = R(2) * mu * E[q] + ((q % 4 == 0) ? lam * trE : R(0));
            frob += E[q] * E[q];
        }
        psi = R(0.5) * lam * trE * trE + mu * frob;
        psip = R(0);
        return 0;
    }
    R w[3], Q[9];
    const int sw = tl::eig3_jacobi(E, w, Q, jtol);
    const R trp = trE > R(0) ? trE : R(0), trm = trE < R(0) ? trE : R(0);
    R pp = R(0.5) * lam * trp * trp, pm = R(0.5) * lam * trm * trm;
    const R s2 = s * s;
    R lp[3], lm[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lp[k] = w[k] > R(0) ? w[k] : R(0);
        lm[k] = w[k] < R(0) ? w[k] : R(0);
        pp += mu * lp[k] * lp[k];
        pm += mu * lm[k] * lm[k];
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            R ep = R(0), em = R(0);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                ep += Q[3 * r + k] * lp[k] * Q[3 * c + k];
                em += Q[3 * r + k] * lm[k] * Q[3 * c + k];
            }
            R sp = R(2) * mu * ep, sm = R(2) * mu * em;
            if (r == c) {
                sp += lam * trp;
                sm += lam * trm;
            }
            S[3 * r + c] = s2 * sp + sm;
        }
    psi = s2 * pp + pm;
    psip = pp;
    return sw >= 64 ? 1 : 0;
}

// J - 1 for F = I + H without cancellation: trH + sum of 2x2 principal minors + det H
template <typename R>
__device__ __forceinline__ R jm1_of(const R* H) {
    const R m2 = (H[0] * H[4] - H[1] * H[3]) + (H[0] * H[8] - H[2] * H[6]) + (H[4] * H[8] - H[5] * H[7]);
    return (H[0] + H[4] + H[8]) + m2 + det3(H);
}

// 0.5*(J^2-1) - ln J for J = 1+e, accurate for small e
template <typename R>
__device__ __forceinline__ R vol_energy_core(R e) {
    if (fabs(e) < R(1e-3)) {
        // e^2 - e^3/3 + e^4/4 - e^5/5 + e^6/6
        return e * e * (R(1) + e * (R(-1) / R(3) + e * (R(0.25) + e * (R(-0.2) + e * (R(1) / R(6))))));
    }
    return e + R(0.5) * e * e - log1p(e);
}

// compressible neo-Hookean through b = F F^T (reference.py:119-148)
template <typename R>
__device__ __forceinline__ int nh_update(const R* H, R kappa, R mu, R s, bool fracture, R* S,
                                         R& psi, R& psip) {
    const R e = jm1_of(H);
    const R J = R(1) + e;
    if (J <= R(TL_J_MIN)) {
#pragma unroll
        for (int q = 0; q < 9; ++q) S[q] = R(0);
        psi = psip = R(0);
        return 1;
    }
    R B[9], b[9], bi[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            B[3 * r + c] = H[3 * r + c] + H[3 * c + r] +
                           (H[3 * r] * H[3 * c] + H[3 * r + 1] * H[3 * c + 1] + H[3 * r + 2] * H[3 * c + 2]);
            b[3 * r + c] = B[3 * r + c] + (r == c ? R(1) : R(0));
        }
    inv3(b, bi);
    const R trB = B[0] + B[4] + B[8];
    // dev(b) = dev(B); I - tr(b)/3 b^-1 = b^-1 dev(B)
    R devB[9], Y[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) devB[q] = B[q] - ((q % 4 == 0) ? trB / R(3) : R(0));
    mm3(bi, devB, Y);
    const R lnJ = log1p(e);
    const R Jm23 = exp(R(-2) / R(3) * lnJ);
    const R Jm23m1 = expm1(R(-2) / R(3) * lnJ);
    const R J2m1 = e * (R(2) + e);
    const R U = R(0.5) * kappa * vol_energy_core(e);
    const R pbar = R(0.5) * mu * (R(3) * Jm23m1 + Jm23 * trB);
    const R s2 = fracture ? s * s : R(1);
    const bool tension = J >= R(1);
    const R wv = tension ? s2 : R(1);
    const R kv = R(0.5) * kappa * J2m1;
#pragma unroll
    for (int q = 0; q < 9; ++q) S[q] = wv * (kv * bi[q]) + s2 * (Jm23 * mu * Y[q]);
    const R pp = tension ? U + pbar : pbar;
    const R pm = tension ? R(0) : U;
    psi = s2 * pp + pm;
    psip = pp;
    return 0;
}

// finite-strain J2 radial return in FP64 on Cp = I + Cpd (reference.py:151-208)
__device__ __forceinline__ int j2_update(const double* F, double* Cpd, double& epb, double mu,
                                         double kappa, double sigma_y0, double H_hard, double* S,
                                         double& psi, double& dwp, bool& nonspd) {
    nonspd = false;
    const double J = det3(F);
    dwp = 0.0;
    if (J <= TL_J_MIN) {
#pragma unroll
        for (int q = 0; q < 9; ++q) S[q] = 0.0;
        psi = 0.0;
        return 1;
    }
    double C[9], Cp[9], Cpi[9], Ce[9], Mdev[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            C[3 * r + c] = F[r] * F[c] + F[3 + r] * F[3 + c] + F[6 + r] * F[6 + c];
    Cp[0] = 1.0 + Cpd[0]; Cp[4] = 1.0 + Cpd[1]; Cp[8] = 1.0 + Cpd[2];
    Cp[1] = Cp[3] = Cpd[3]; Cp[2] = Cp[6] = Cpd[4]; Cp[5] = Cp[7] = Cpd[5];
    inv3(Cp, Cpi);
    mm3(C, Cpi, Ce);
    const double fac = pow(J, -2.0 / 3.0);
    const double tr3 = fac * (Ce[0] + Ce[4] + Ce[8]) / 3.0;
    double frob = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        Mdev[q] = mu * (fac * Ce[q] - ((q % 4 == 0) ? tr3 : 0.0));
        frob += Mdev[q] * Mdev[q];
    }
    const double sigeq = sqrt(1.5 * frob);
    const double sy = sigma_y0 + H_hard * epb;
    if (sigeq - sy > 0.0) {
        const double sq23 = sqrt(2.0 / 3.0);
        const double dg = (sigeq - sy) / (3.0 * mu + H_hard * sq23);
        const double scale = 1.0 - 3.0 * mu * dg / sigeq;
        double N[9], NC[9], Cn[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) N[q] = (1.5 / sigeq) * Mdev[q];
        mm3(N, Cp, NC);
#pragma unroll
        for (int q = 0; q < 9; ++q) Cn[q] = Cp[q] + 2.0 * dg * NC[q];
        Cn[1] = Cn[3] = 0.5 * (Cn[1] + Cn[3]);
        Cn[2] = Cn[6] = 0.5 * (Cn[2] + Cn[6]);
        Cn[5] = Cn[7] = 0.5 * (Cn[5] + Cn[7]);
        const double dC = det3(Cn);
        if (dC <= 0.0) {
            nonspd = true;
            return 0;
        }
        const double proj = pow(dC, -1.0 / 3.0);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            Cp[q] = Cn[q] * proj;
            Mdev[q] *= scale;
        }
        Cpd[0] = Cp[0] - 1.0; Cpd[1] = Cp[4] - 1.0; Cpd[2] = Cp[8] - 1.0;
        Cpd[3] = Cp[1]; Cpd[4] = Cp[2]; Cpd[5] = Cp[5];
        const double deb = sq23 * dg;
        dwp = (sy + 0.5 * H_hard * deb) * deb;
        epb += deb;
        inv3(Cp, Cpi);
        mm3(C, Cpi, Ce);
    }
    double Cei[9], Ci[9], T[9], Sd[9];
    inv3(Ce, Cei);
    inv3(C, Ci);
    mm3(Cei, Mdev, T);
    mm3(T, Cei, Sd);
    const double vol = 0.5 * kappa * (J * J - 1.0);
#pragma unroll
    for (int q = 0; q < 9; ++q) S[q] = Sd[q] / J + vol * Ci[q];
    S[1] = S[3] = 0.5 * (S[1] + S[3]);
    S[2] = S[6] = 0.5 * (S[2] + S[6]);
    S[5] = S[7] = 0.5 * (S[5] + S[7]);
    const double trbar = fac * (Ce[0] + Ce[4] + Ce[8]);
    psi = 0.25 * kappa * (J * J - 1.0 - 2.0 * log(J)) + 0.5 * mu * (trbar - 3.0);
    return 0;
}

template <typename R>
__device__ __forceinline__ R planeR(const void* p, int64_t stride, int c, int64_t i) {
    return static_cast<const R*>(p)[c * stride + i];
}

// ---------------------------------------------------------------------------
// pass A
// ---------------------------------------------------------------------------
template <typename R, int DIM, int MODEL, bool FRAC>
__global__ void __launch_bounds__(kThreads) k_pass_a(const tl_body b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    __shared__ double s_pw[kThreads / 32];
    double pw = 0.0;
    if (halted(b)) return;
    if (i < b.n) {
        const int64_t N = b.n_all;
        const R* us = static_cast<const R*>(b.us);
        const int lane = (int)(i & 31);
        const int64_t w = i >> 5;
        const int64_t base = b.soff[w];
        const int len = (int)((b.soff[w + 1] - base) >> 5);
        const double xi = b.Xs[i], yi = b.Xs[N + i], zi = b.Xs[2 * N + i];
        const auto ui = tl::ld4(us + 4 * i);
        const R si = ui.w;
        const bool gated = FRAC && si <= R(b.s_l);
        const R inv_h = R(b.inv_h), alpha = R(b.alpha);
        R D[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) D[q] = R(0);
        R M[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};   // xx yy zz xy xz yz
        const int32_t* sidx = b.sidx + base + lane;
        for (int k = 0; k < len; ++k) {
            const int32_t j = __ldg(sidx + 32 * k);
            if (j < 0) break;
            const R dx = R(xi - __ldg(b.Xs + j));
            const R dy = DIM == 3 ? R(yi - __ldg(b.Xs + N + j)) : R(0);
            const R dz = R(zi - __ldg(b.Xs + 2 * N + j));
            const R r2 = dx * dx + dy * dy + dz * dz;
            const R r = sqrt(r2);
            const R fac = tl::kernel_fac(r, inv_h, alpha, b.kind);
            const auto uj = tl::ldg4(us + 4 * (int64_t)j);
            const R vj = b.uniform ? R(b.V0c) : R(b.V0[j]);
            const R wf = vj * fac;
            if (!gated) {
                const R du0 = wf * (uj.x - ui.x), du2 = wf * (uj.z - ui.z);
                D[0] += du0 * dx; D[2] += du0 * dz;
                D[6] += du2 * dx; D[8] += du2 * dz;
                if (DIM == 3) {
                    const R du1 = wf * (uj.y - ui.y);
                    D[1] += du0 * dy; D[7] += du2 * dy;
                    D[3] += du1 * dx; D[4] += du1 * dy; D[5] += du1 * dz;
                }
            }
            if (FRAC) {
                const R c = r2 > R(0) ? R(2) * (si - uj.w) * wf / r2 : R(0);
                const R cx = c * dx, cz = c * dz;
                M[0] += cx * dx; M[2] += cz * dz; M[4] += cx * dz;
                if (DIM == 3) {
                    const R cy = c * dy;
                    M[1] += cy * dy; M[3] += cx * dy; M[5] += cy * dz;
                }
            }
        }
        // L_i (9 planes)
        R Li[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) Li[q] = planeR<R>(b.L, N, q, i);
        // H = F - I = D L^T
        R Hm[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                Hm[3 * r + c] = D[3 * r] * Li[3 * c] + D[3 * r + 1] * Li[3 * c + 1] + D[3 * r + 2] * Li[3 * c + 2];
        if (gated) {
#pragma unroll
            for (int q = 0; q < 9; ++q) Hm[q] = R(0);
        }
        // constitutive update
        R S[9], psi = R(0), psip = R(0);
        int bad = 0, noconv = 0;
        if (MODEL == 1) {
            noconv = svk_update<R>(Hm, R(b.lam), R(b.mu), si, FRAC, R(b.jac_tol), S, psi, psip);
        } else if (MODEL == 2) {
            bad = nh_update<R>(Hm, R(b.kappa), R(b.mu), si, FRAC, S, psi, psip);
        } else {
            double Fd[9], Cpd[6], Sd[9], psid, dwp;
            bool nonspd;
#pragma unroll
            for (int q = 0; q < 9; ++q) Fd[q] = double(Hm[q]) + ((q % 4 == 0) ? 1.0 : 0.0);
#pragma unroll
            for (int q = 0; q < 6; ++q) Cpd[q] = double(planeR<R>(b.Cpd, N, q, i));
            double epb = double(static_cast<const R*>(b.epbar)[i]);
            bad = j2_update(Fd, Cpd, epb, b.mu, b.kappa, b.sigma_y0, b.H_hard, Sd, psid, dwp, nonspd);
            if (nonspd) atomicMin((long long*)&b.counters[2], (long long)i);
#pragma unroll
            for (int q = 0; q < 6; ++q) static_cast<R*>(b.Cpd)[q * N + i] = R(Cpd[q]);
            static_cast<R*>(b.epbar)[i] = R(epb);
#pragma unroll
            for (int q = 0; q < 9; ++q) S[q] = R(Sd[q]);
            psi = R(psid);
            psip = R(0);
            pw = dwp * (b.uniform ? b.V0c : b.V0[i]);
        }
        // phase field: history, Laplacian, s-ddot (fracture.py:12-43)
        if (FRAC) {
            R* Hh = static_cast<R*>(b.Hh);
            const R Hn = fmax(psip, Hh[i]);
            Hh[i] = Hn;
            const R lap = Li[0] * M[0] + Li[4] * M[1] + Li[8] * M[2] + (Li[1] + Li[3]) * M[3] +
                          (Li[2] + Li[6]) * M[4] + (Li[5] + Li[7]) * M[5];
            const R eps0 = R(b.eps0), Gc = R(b.Gc), c0 = R(b.c0);
            const R ratio = Hn / Gc;
            const R damp = R(2) * sqrt(R(4) * eps0 * ratio + R(1)) / c0;
            const R sd = static_cast<const R*>(b.sdot)[i];
            static_cast<R*>(b.sddot)[i] =
                (c0 * c0 / (R(2) * eps0)) *
                (R(2) * eps0 * lap + (R(1) - si) / (R(2) * eps0) - damp * sd - R(2) * si * ratio);
        }
        // P = F S = S + H S ; PL = P L_i
        R P[9], PL[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                P[3 * r + c] = S[3 * r + c] + (Hm[3 * r] * S[c] + Hm[3 * r + 1] * S[3 + c] + Hm[3 * r + 2] * S[6 + c]);
        mm3(P, Li, PL);
        // viscosity tensor: det(F) F^-1 = adj(F), zero when det F <= J_MIN
        R* al = static_cast<R*>(b.al);
        if (b.visc) {
            R Fm[9], A[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) Fm[q] = Hm[q] + ((q % 4 == 0) ? R(1) : R(0));
            const R J = R(1) + jm1_of(Hm);
            if (J > R(TL_J_MIN)) {
                R adj[9];
                adj[0] = Fm[4] * Fm[8] - Fm[5] * Fm[7];
                adj[1] = Fm[2] * Fm[7] - Fm[1] * Fm[8];
                adj[2] = Fm[1] * Fm[5] - Fm[2] * Fm[4];
                adj[3] = Fm[5] * Fm[6] - Fm[3] * Fm[8];
                adj[4] = Fm[0] * Fm[8] - Fm[2] * Fm[6];
                adj[5] = Fm[2] * Fm[3] - Fm[0] * Fm[5];
                adj[6] = Fm[3] * Fm[7] - Fm[4] * Fm[6];
                adj[7] = Fm[1] * Fm[6] - Fm[0] * Fm[7];
                adj[8] = Fm[0] * Fm[4] - Fm[1] * Fm[3];
                mm3(adj, Li, A);
            } else {
#pragma unroll
                for (int q = 0; q < 9; ++q) A[q] = R(0);
                bad += 1;
            }
#pragma unroll
            for (int q = 0; q < 9; ++q) al[q * N + i] = A[q];
        }
        // pass-B gather record: PL (9) + v (3)
        const R* vv = static_cast<const R*>(b.v);
        R* rb = static_cast<R*>(b.rb) + 12 * i;
        tl::st4(rb, PL[0], PL[1], PL[2], PL[3]);
        tl::st4(rb + 4, PL[4], PL[5], PL[6], PL[7]);
        tl::st4(rb + 8, PL[8], vv[i], vv[N + i], vv[2 * N + i]);
        if (mirror_out(b)) {
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                b.F_out[9 * i + q] = double(Hm[q]) + ((q % 4 == 0) ? 1.0 : 0.0);
                b.S_out[9 * i + q] = double(S[q]);
            }
            b.psi_out[i] = double(psi);
            b.psip_out[i] = double(psip);
        }
        if (bad || noconv) {
            if (bad) atomicAdd((unsigned long long*)&b.counters[0], (unsigned long long)bad);
            if (noconv) atomicAdd((unsigned long long*)&b.counters[1], 1ull);
        }
    }
    if (MODEL == 3) {
        // deterministic block partial of sum(dwp * V0)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
        if ((threadIdx.x & 31) == 0) s_pw[threadIdx.x >> 5] = pw;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int k = 0; k < kThreads / 32; ++k) t += s_pw[k];
            b.pw_partial[blockIdx.x] = t;
        }
    }
}

// ---------------------------------------------------------------------------
// boundary conditions (dynamics.py:159-217, fracture.py:46-83)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void make_vars(tl::ExprVars& V, double x0, double y0, double z0,
                                          double ux, double uy, double uz, double t, double dt,
                                          double dx) {
    V.v[0] = x0; V.v[1] = y0; V.v[2] = z0;
    V.v[3] = x0 + ux; V.v[4] = y0 + uy; V.v[5] = z0 + uz;
    V.v[6] = ux; V.v[7] = uy; V.v[8] = uz;
    V.v[9] = t; V.v[10] = dt; V.v[11] = dx;
}

// the slice of tl_body the boundary-condition code needs, passed by value so
// out-of-line calls never copy the whole descriptor to local memory
struct BcCtx {
    const tl_bc* bcs;
    const tl_prog* progs;
    int64_t* counters;
    double dp_body;
    int nbc, dim, restrict_prog;
};

__device__ __forceinline__ BcCtx bc_ctx(const tl_body& b) {
    return BcCtx{b.bcs, b.progs, b.counters, b.dp_body, b.nbc, b.dim, b.restrict_prog};
}

__device__ __forceinline__ void note_err(const BcCtx& b, int err) {
    if (err) atomicCAS((unsigned long long*)&b.counters[4], 0ull, (unsigned long long)err);
}

__device__ __forceinline__ bool bc_applies(const tl_bc& c, uint32_t mask, double t) {
    if (!(c.tst <= t && t <= c.tend)) return false;
    return c.bit < 0 || ((mask >> c.bit) & 1u);
}

// add force BCs active at t to acc (in file order).  Out of line so the
// evaluator's stack frame never competes with the gather loop's registers.
__device__ __noinline__ void force_bcs(const BcCtx b, uint32_t mask, double m0i, const tl::ExprVars& V,
                          double t, double* acc) {
    for (int k = 0; k < b.nbc; ++k) {
        const tl_bc c = b.bcs[k];
        if (c.kind != 1 || !bc_applies(c, mask, t)) continue;
        double scale = 1.0;
        if (c.ftype == 1) scale = 1.0 / m0i;
        else if (c.ftype == 2) scale = (b.dim == 3 ? b.dp_body * b.dp_body : b.dp_body) / m0i;
        for (int ax = 0; ax < 3; ++ax) {
            if (c.has_const[ax]) {
                acc[ax] = tl::add_rn(acc[ax], tl::mul_rn(c.cval[ax], scale));
            } else if (c.prog[ax] >= 0) {
                bool skip;
                int err = 0;
                const double val = tl::expr_eval(b.progs[c.prog[ax]], V, &skip, &err);
                note_err(b, err);
                acc[ax] = tl::add_rn(acc[ax], skip ? 0.0 : tl::mul_rn(val, scale));
            }
        }
    }
}

// overwrite velocity components from velocity BCs active at t (file order)
__device__ __noinline__ void velocity_bcs(const BcCtx b, uint32_t mask, const tl::ExprVars& V, double t,
                             double* vel) {
    for (int k = 0; k < b.nbc; ++k) {
        const tl_bc c = b.bcs[k];
        if (c.kind != 0 || !bc_applies(c, mask, t)) continue;
        for (int ax = 0; ax < 3; ++ax) {
            if (c.has_const[ax]) {
                vel[ax] = c.cval[ax];
            } else if (c.prog[ax] >= 0) {
                bool skip;
                int err = 0;
                const double val = tl::expr_eval(b.progs[c.prog[ax]], V, &skip, &err);
                note_err(b, err);
                if (!skip) vel[ax] = val;
            }
        }
    }
    if (b.dim == 2) vel[1] = 0.0;
}

// sdot += dtr*sddot; s += dts*sdot; clamp [0,1]; restrictphi floor
template <typename R>
__device__ __forceinline__ void advance_phase(const BcCtx& b, R& s, R& sd, R sdd, double dts,
                                              double dtr, const tl::ExprVars& V) {
    sd = tl::axpy_rn(sd, R(dtr), sdd);
    s = tl::axpy_rn(s, R(dts), sd);
    if (s < R(0)) { s = R(0); sd = R(0); }
    if (s > R(1)) { s = R(1); sd = R(0); }
    if (b.restrict_prog >= 0) {
        bool skip;
        int err = 0;
        const double val = tl::expr_eval(b.progs[b.restrict_prog], V, &skip, &err);
        note_err(b, err);
        if (!skip) {
            if (val < 0.0 || val > 1.0) atomicExch((unsigned long long*)&b.counters[5], 1ull);
            if (double(s) < val) {
                s = R(val);
                sd = R(0);
            }
        }
    }
}

__device__ __forceinline__ double sq3_rn(double x, double y, double z) {
    // numpy einsum("nd,nd->n") order on (n,3): (x*x + z*z) + y*y
    return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(z, z)), __dmul_rn(y, y));
}

// ---------------------------------------------------------------------------
// pass B
// ---------------------------------------------------------------------------
template <typename R, int DIM, int MODE, bool FRAC>
__global__ void __launch_bounds__(kThreads) k_pass_b(const tl_body b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (halted(b)) return;
    double v2 = 0.0, a2 = 0.0;
    long long bad_acc = LLONG_MAX;
    if (i < b.n) {
        const int64_t N = b.n_all;
        const R* rbp = static_cast<const R*>(b.rb);
        const int lane = (int)(i & 31);
        const int64_t w = i >> 5;
        const int64_t base = b.soff[w];
        const int len = (int)((b.soff[w + 1] - base) >> 5);
        const double xi = b.Xs[i], yi = b.Xs[N + i], zi = b.Xs[2 * N + i];
        const auto r0i = tl::ld4(rbp + 12 * i);
        const auto r1i = tl::ld4(rbp + 12 * i + 4);
        const auto r2i = tl::ld4(rbp + 12 * i + 8);
        const R vi0 = r2i.y, vi1 = r2i.z, vi2 = r2i.w;
        const R inv_h = R(b.inv_h), alpha = R(b.alpha);
        const bool visc = b.visc != 0;
        const R eps_h2 = R(0.001 * b.h * b.h);
        const R hR = R(b.h), b1c0 = R(b.beta1 * b.c0), b2 = R(b.beta2), inv_rho = R(1.0 / b.rho0);
        R s1[3] = {R(0), R(0), R(0)}, s2[3] = {R(0), R(0), R(0)}, s3[3] = {R(0), R(0), R(0)};
        const int32_t* sidx = b.sidx + base + lane;
        for (int k = 0; k < len; ++k) {
            const int32_t j = __ldg(sidx + 32 * k);
            if (j < 0) break;
            const R dx = R(xi - __ldg(b.Xs + j));
            const R dy = DIM == 3 ? R(yi - __ldg(b.Xs + N + j)) : R(0);
            const R dz = R(zi - __ldg(b.Xs + 2 * N + j));
            const R r2 = dx * dx + dy * dy + dz * dz;
            const R fac = tl::kernel_fac(sqrt(r2), inv_h, alpha, b.kind);
            const R* rj = rbp + 12 * (int64_t)j;
            const auto q0 = tl::ldg4(rj);
            const auto q1 = tl::ldg4(rj + 4);
            const auto q2 = tl::ldg4(rj + 8);
            const R mj = b.uniform ? R(b.m0c) : R(b.m0[j]);
            const R wf = mj * fac;
            // PL_j r0 (row-major PL_j = q0.x..q2.x)
            R p0, p1, p2;
            if (DIM == 3) {
                p0 = q0.x * dx + q0.y * dy + q0.z * dz;
                p1 = q0.w * dx + q1.x * dy + q1.y * dz;
                p2 = q1.z * dx + q1.w * dy + q2.x * dz;
            } else {
                p0 = q0.x * dx + q0.z * dz;
                p1 = R(0);
                p2 = q1.z * dx + q2.x * dz;
            }
            s1[0] += wf * dx; s1[2] += wf * dz;
            s2[0] += wf * p0; s2[2] += wf * p2;
            if (DIM == 3) {
                s1[1] += wf * dy;
                s2[1] += wf * p1;
            }
            if (visc) {
                const R dvr = (vi0 - q2.y) * dx + (DIM == 3 ? (vi1 - q2.z) * dy : R(0)) + (vi2 - q2.w) * dz;
                const R G = hR * dvr / (r2 + eps_h2);
                const R pw = (b2 * G * G - b1c0 * G) * inv_rho * wf;
                s3[0] += pw * dx; s3[2] += pw * dz;
                if (DIM == 3) s3[1] += pw * dy;
            }
        }
        // a_int = (PL_i s1 + s2)/rho0^2 - AL_i s3
        const R PLi[9] = {r0i.x, r0i.y, r0i.z, r0i.w, r1i.x, r1i.y, r1i.z, r1i.w, r2i.x};
        const R inv_rho2 = inv_rho * inv_rho;
        double acc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            R t = (PLi[3 * a] * s1[0] + PLi[3 * a + 1] * s1[1] + PLi[3 * a + 2] * s1[2] + s2[a]) * inv_rho2;
            if (visc) {
                const R* al = static_cast<const R*>(b.al);
                t -= al[(3 * a) * N + i] * s3[0] + al[(3 * a + 1) * N + i] * s3[1] +
                     al[(3 * a + 2) * N + i] * s3[2];
            }
            acc[a] = double(t);
        }
        // a = a_int + f0 + force BCs ; 2D a_y = 0  (stepper.py:86-95)
        acc[0] = tl::add_rn(acc[0], b.f0[0]);
        acc[1] = tl::add_rn(acc[1], b.f0[1]);
        acc[2] = tl::add_rn(acc[2], b.f0[2]);
        const R* us = static_cast<const R*>(b.us);
        const auto ui = tl::ld4(us + 4 * i);
        const uint32_t mask = b.bcmask ? b.bcmask[i] : 0u;
        const double t0 = b.clock ? b.clock->t : 0.0;
        const double dt = b.clock ? b.clock->dt : 0.0;
        tl::ExprVars V;
        const double m0i = b.uniform ? b.m0c : b.m0[i];
        const double tf = MODE == TL_B_INIT ? 0.0 : (MODE == TL_B_SYMPL ? t0 + 0.5 * dt : t0);
        const double dtf = MODE == TL_B_INIT ? 0.0 : dt;
        make_vars(V, xi, yi, zi, double(ui.x), double(ui.y), double(ui.z), tf, dtf, b.dp_body);
        if (b.nbc && (mask || b.bc_whole)) force_bcs(bc_ctx(b), mask, m0i, V, tf, acc);
        if (DIM == 2) acc[1] = 0.0;
        if (!(isfinite(acc[0]) && isfinite(acc[1]) && isfinite(acc[2]))) {
            bad_acc = (long long)i;
            if (b.clock) atomicMin((long long*)&b.counters[6], (long long)b.clock->step);
        }
        // velocity: v_i is the copy pass A put in the record
        double vel[3] = {double(vi0), double(vi1), double(vi2)};
        R us_new[4] = {ui.x, ui.y, ui.z, ui.w};
        R* vout = static_cast<R*>(b.v);
        if (MODE == TL_B_INIT) {
            if (b.nbc && (mask || b.bc_whole)) velocity_bcs(bc_ctx(b), mask, V, 0.0, vel);
        } else {
            const double kick = MODE == TL_B_VERLET ? dt : 0.5 * dt;
            const double t_new = t0 + dt;
            // BC phase at the force time, kick, BCs at t_new, drift
            if (b.nbc && (mask || b.bc_whole)) velocity_bcs(bc_ctx(b), mask, V, tf, vel);
            R vR[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) vR[a] = tl::axpy_rn(R(vel[a]), R(kick), R(acc[a]));
#pragma unroll
            for (int a = 0; a < 3; ++a) vel[a] = double(vR[a]);
            V.v[9] = t_new;
            if (b.nbc && (mask || b.bc_whole)) velocity_bcs(bc_ctx(b), mask, V, t_new, vel);
#pragma unroll
            for (int a = 0; a < 3; ++a) vR[a] = R(vel[a]);
            us_new[0] = tl::axpy_rn(ui.x, R(kick), vR[0]);
            us_new[1] = DIM == 3 ? tl::axpy_rn(ui.y, R(kick), vR[1]) : R(0);
            us_new[2] = tl::axpy_rn(ui.z, R(kick), vR[2]);
            if (FRAC) {
                R* sdp = static_cast<R*>(b.sdot);
                R sd = sdp[i];
                R s = ui.w;
                const R sdd = static_cast<const R*>(b.sddot)[i];
                tl::ExprVars Vn;
                make_vars(Vn, xi, yi, zi, double(us_new[0]), double(us_new[1]), double(us_new[2]),
                          t_new, dt, b.dp_body);
                advance_phase<R>(bc_ctx(b), s, sd, sdd, kick, kick, Vn);
                us_new[3] = s;
                sdp[i] = sd;
            }
            tl::st4(static_cast<R*>(b.us) + 4 * i, us_new[0], us_new[1], us_new[2], us_new[3]);
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) vout[a * N + i] = R(vel[a]);
        if (b.store_a || mirror_out(b)) {
            R* ap = static_cast<R*>(b.a);
#pragma unroll
            for (int a = 0; a < 3; ++a) ap[a * N + i] = R(acc[a]);
        }
        if (MODE != TL_B_INIT && b.clock &&
            !(isfinite(vel[0]) && isfinite(vel[1]) && isfinite(vel[2]) && isfinite(double(us_new[0])) &&
              isfinite(double(us_new[1])) && isfinite(double(us_new[2]))))
            atomicMin((long long*)&b.counters[7], (long long)b.clock->step + 1);
        const double vx = double(R(vel[0])), vy = double(R(vel[1])), vz = double(R(vel[2]));
        const double ax = double(R(acc[0])), ay = double(R(acc[1])), az = double(R(acc[2]));
        v2 = sq3_rn(vx, vy, vz);
        a2 = sq3_rn(ax, ay, az);
        if (!(a2 == a2)) a2 = 0.0;  // NaN is reported through counters[3]
    }
    v2 = tl::warp_max(v2);
    a2 = tl::warp_max(a2);
    bad_acc = tl::warp_min_ll(bad_acc);
    if ((threadIdx.x & 31) == 0) {
        tl::atomic_max_nonneg(&b.red[0], v2);
        tl::atomic_max_nonneg(&b.red[1], a2);
        if (bad_acc != LLONG_MAX) atomicMin((long long*)&b.counters[3], bad_acc);
    }
}

// symplectic predictor (stepper.py:168-175)
template <typename R, int DIM, bool FRAC>
__global__ void __launch_bounds__(kThreads) k_predict(const tl_body b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (halted(b) || i >= b.n) return;
    const int64_t N = b.n_all;
    const double t0 = b.clock->t, dt = b.clock->dt;
    const double th = t0 + 0.5 * dt;
    const double half = 0.5 * dt;
    R* vp = static_cast<R*>(b.v);
    const R* ap = static_cast<const R*>(b.a);
    R* us = static_cast<R*>(b.us);
    const auto ui = tl::ld4(us + 4 * i);
    const double xi = b.Xs[i], yi = b.Xs[N + i], zi = b.Xs[2 * N + i];
    double vel[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) vel[a] = double(tl::axpy_rn(vp[a * N + i], R(half), ap[a * N + i]));
    const uint32_t mask = b.bcmask ? b.bcmask[i] : 0u;
    tl::ExprVars V;
    make_vars(V, xi, yi, zi, double(ui.x), double(ui.y), double(ui.z), th, dt, b.dp_body);
    if (b.nbc && (mask || b.bc_whole)) velocity_bcs(bc_ctx(b), mask, V, th, vel);
    R vR[3] = {R(vel[0]), R(vel[1]), R(vel[2])};
    R un[4] = {tl::axpy_rn(ui.x, R(half), vR[0]), DIM == 3 ? tl::axpy_rn(ui.y, R(half), vR[1]) : R(0),
               tl::axpy_rn(ui.z, R(half), vR[2]), ui.w};
    if (FRAC) {
        R* sdp = static_cast<R*>(b.sdot);
        R sd = sdp[i], s = ui.w;
        tl::ExprVars Vn;
        make_vars(Vn, xi, yi, zi, double(un[0]), double(un[1]), double(un[2]), th, dt, b.dp_body);
        advance_phase<R>(bc_ctx(b), s, sd, static_cast<const R*>(b.sddot)[i], half, half, Vn);
        un[3] = s;
        sdp[i] = sd;
    }
    tl::st4(us + 4 * i, un[0], un[1], un[2], un[3]);
#pragma unroll
    for (int a = 0; a < 3; ++a) vp[a * N + i] = vR[a];
}

// ---------------------------------------------------------------------------
// device clock (stepper.py:19-25, 199-263)
// ---------------------------------------------------------------------------
struct DtInfos {
    tl_dtinfo d[8];
    int n;
};

__global__ void k_clock_begin(tl_clock* c, DtInfos info) {
    if (c->halted) return;
    if (!(c->t < c->t_max - c->eps)) {
        c->halted = 1;
        return;
    }
    double dt;
    if (c->dt_override >= 0.0) {
        dt = c->dt_override;
    } else {
        dt = INFINITY;
        for (int k = 0; k < info.n; ++k) {
            const double vmax = sqrt(__longlong_as_double((long long)info.d[k].red[0]));
            const double amax = sqrt(__longlong_as_double((long long)info.d[k].red[1]));
            const double dtv = info.d[k].h / (info.d[k].c0 + vmax);
            double cand = amax > 0.0 ? c->cfl * fmin(dtv, sqrt(info.d[k].h / amax)) : c->cfl * dtv;
            dt = fmin(dt, cand);
        }
    }
    dt = fmin(fmin(dt, c->next_out - c->t), c->t_max - c->t);
    if (!(dt > 0.0)) {
        c->halted = 4;
        c->dt = dt;
        return;
    }
    c->dt = dt;
    const double tn = c->t + dt;
    c->out_step = (tn >= c->next_out - c->eps) || (tn >= c->t_max - c->eps) ||
                  (c->max_steps >= 0 && c->step + 1 >= c->max_steps);
}

__global__ void k_clock_commit(tl_clock* c) {
    if (c->halted) return;
    c->t += c->dt;
    c->step += 1;
    if (c->t >= c->next_out - c->eps) c->halted = 2;
    else if (c->max_steps >= 0 && c->step >= c->max_steps) c->halted = 3;
}

__global__ void k_reduce_partials(const double* p, int64_t n, double* acc) {
    __shared__ double s[1024];
    double t = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) t += p[k];
    s[threadIdx.x] = t;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *acc += s[0];
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
template <typename R, int DIM>
int launch_a(cudaStream_t st, const tl_body& b) {
    const unsigned g = tl_blocks(b.n, kThreads);
    if (b.model == 1) {
        if (b.fracture) k_pass_a<R, DIM, 1, true><<<g, kThreads, 0, st>>>(b);
        else k_pass_a<R, DIM, 1, false><<<g, kThreads, 0, st>>>(b);
    } else if (b.model == 2) {
        if (b.fracture) k_pass_a<R, DIM, 2, true><<<g, kThreads, 0, st>>>(b);
        else k_pass_a<R, DIM, 2, false><<<g, kThreads, 0, st>>>(b);
    } else {
        k_pass_a<R, DIM, 3, false><<<g, kThreads, 0, st>>>(b);
    }
    return tl_check_launch("k_pass_a");
}

template <typename R, int DIM, int MODE>
int launch_b_mode(cudaStream_t st, const tl_body& b) {
    const unsigned g = tl_blocks(b.n, kThreads);
    if (b.fracture) k_pass_b<R, DIM, MODE, true><<<g, kThreads, 0, st>>>(b);
    else k_pass_b<R, DIM, MODE, false><<<g, kThreads, 0, st>>>(b);
    return tl_check_launch("k_pass_b");
}

template <typename R, int DIM>
int launch_b(cudaStream_t st, const tl_body& b, int mode) {
    if (mode == TL_B_INIT) return launch_b_mode<R, DIM, TL_B_INIT>(st, b);
    if (mode == TL_B_VERLET) return launch_b_mode<R, DIM, TL_B_VERLET>(st, b);
    return launch_b_mode<R, DIM, TL_B_SYMPL>(st, b);
}

template <typename R, int DIM>
int launch_p(cudaStream_t st, const tl_body& b) {
    const unsigned g = tl_blocks(b.n, kThreads);
    if (b.fracture) k_predict<R, DIM, true><<<g, kThreads, 0, st>>>(b);
    else k_predict<R, DIM, false><<<g, kThreads, 0, st>>>(b);
    return tl_check_launch("k_predict");
}

int check_body(const tl_body* b) {
    if (!b || b->n <= 0 || (b->precision != 4 && b->precision != 8) || (b->dim != 2 && b->dim != 3) ||
        b->model < 1 || b->model > 3 || !b->soff || !b->sidx || !b->Xs || !b->us || !b->rb) {
        tl_set_error("tl_body: invalid descriptor");
        return TL_ERR_ARG;
    }
    return TL_OK;
}

}  // namespace

extern "C" int64_t tl_pass_blocks(int64_t n) { return (int64_t)tl_blocks(n, kThreads); }

extern "C" int tl_pass_a(tl_stream_t st_, const tl_body* b) {
    int rc = check_body(b);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)st_;
    if (b->precision == 4) return b->dim == 3 ? launch_a<float, 3>(st, *b) : launch_a<float, 2>(st, *b);
    return b->dim == 3 ? launch_a<double, 3>(st, *b) : launch_a<double, 2>(st, *b);
}

extern "C" int tl_pass_b(tl_stream_t st_, const tl_body* b, int mode) {
    int rc = check_body(b);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)st_;
    if (b->precision == 4)
        return b->dim == 3 ? launch_b<float, 3>(st, *b, mode) : launch_b<float, 2>(st, *b, mode);
    return b->dim == 3 ? launch_b<double, 3>(st, *b, mode) : launch_b<double, 2>(st, *b, mode);
}

extern "C" int tl_predict(tl_stream_t st_, const tl_body* b) {
    int rc = check_body(b);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)st_;
    if (b->precision == 4) return b->dim == 3 ? launch_p<float, 3>(st, *b) : launch_p<float, 2>(st, *b);
    return b->dim == 3 ? launch_p<double, 3>(st, *b) : launch_p<double, 2>(st, *b);
}

extern "C" int tl_clock_begin(tl_stream_t st, tl_clock* clock, int nbody, const tl_dtinfo* info) {
    if (nbody < 0 || nbody > 8) {
        tl_set_error("tl_clock_begin: at most 8 bodies");
        return TL_ERR_ARG;
    }
    DtInfos d;
    d.n = nbody;
    for (int k = 0; k < nbody; ++k) d.d[k] = info[k];
    k_clock_begin<<<1, 1, 0, (cudaStream_t)st>>>(clock, d);
    return tl_check_launch("k_clock_begin");
}

extern "C" int tl_clock_commit(tl_stream_t st, tl_clock* clock) {
    k_clock_commit<<<1, 1, 0, (cudaStream_t)st>>>(clock);
    return tl_check_launch("k_clock_commit");
}

extern "C" int tl_reset_red(tl_stream_t st, unsigned long long* red) {
    TL_TRY_CUDA(cudaMemsetAsync(red, 0, 2 * sizeof(unsigned long long), (cudaStream_t)st));
    return TL_OK;
}

extern "C" int tl_reduce_partials(tl_stream_t st, const double* partials, int64_t nparts,
                                  double* acc) {
    if (nparts <= 0) return TL_OK;
    k_reduce_partials<<<1, 1024, 0, (cudaStream_t)st>>>(partials, nparts, acc);
    return tl_check_launch("k_reduce_partials");
}
