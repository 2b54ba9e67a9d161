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
#include <type_traits>

#include "expr_vm.cuh"
#include "tl_common.cuh"

namespace {

using tl::det3;
using tl::inv3;
using tl::mm3;

#ifndef TL_THREADS
#define TL_THREADS 256
#endif
// neighbours gathered per group (must divide TL_SELL_GROUP)
#ifndef TL_GATHER_A
#define TL_GATHER_A 4
#endif
#ifndef TL_GATHER_B
#define TL_GATHER_B 4
#endif
// minimum resident CTAs per SM requested from ptxas (register budget, for
// 256-thread launch bounds); tuned on B200 for the C4 workload: FP32 pass A
// and pass B 4 (64 registers; 48 spills and measured slower); FP64 2 (128
// registers: 64 spilled 2 KB in pass B, 136 in pass A left it at 3 CTAs/SM)
#ifndef TL_MINB_A_GATHER
#define TL_MINB_A_GATHER 3
#endif
#ifndef TL_MINB_A
#ifndef TL_MINB_A_F64
#define TL_MINB_A_F64 2
#endif
#define TL_MINB_A(R, TILED) (sizeof(R) == 4 ? ((TILED) ? 4 : TL_MINB_A_GATHER) : TL_MINB_A_F64)
#endif
#ifndef TL_MINB_B
#ifndef TL_MINB_B_F32
#define TL_MINB_B_F32 4
#endif
#ifndef TL_MINB_B_F64
#define TL_MINB_B_F64 2
#endif
#define TL_MINB_B(R) (sizeof(R) == 4 ? TL_MINB_B_F32 : TL_MINB_B_F64)
#endif
static_assert(TL_SELL_GROUP % TL_GATHER_A == 0 && TL_SELL_GROUP % TL_GATHER_B == 0, "gather group");
static_assert(TL_SELL_GROUP == 4, "tiled neighbour loops read 4 slots per group");
constexpr int kThreads = TL_THREADS;

__device__ __forceinline__ bool halted(const tl_body& b) {
    return b.clock != nullptr && *(volatile int32_t*)&b.clock->halted != 0;
}

// a stress error of this step (eigen non-convergence, non-SPD plastic
// metric): the reference raises it inside update_stress, before momentum
// and the kick (constitutive.py:177-194), so pass B does nothing
__device__ __forceinline__ bool stress_failed(const tl_body& b) {
    return b.clock != nullptr && (*(volatile int32_t*)&b.clock->err & 1);
}

// an error the reference raises inside the step: the clock does not commit
// the step and halts at the next begin
__device__ __forceinline__ void flag_step_error(tl_clock* c, int bit) {
    if (c != nullptr) atomicOr(&c->err, bit);
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

// Positive part E+ of a symmetric 3x3 E (E- = E - E+), FP32 mode.
// Closed form instead of Jacobi sweeps: eigenvalues by the trigonometric
// (Cardano) method, then the projector of the one eigenvalue whose sign
// differs from the other two (Sylvester: P_k = prod_{j!=k} (E - l_j I) /
// (l_k - l_j)).  Its denominators are bounded below by |l_k| > 0, so the
// split is well conditioned even when the two same-sign eigenvalues are
// (nearly) equal -- the case where individual eigenvectors are not.
// Symmetric storage e = (xx, yy, zz, xy, xz, yz).
__device__ __forceinline__ void positive_part_sym(const float* e, float* ep) {
    const float q = (e[0] + e[1] + e[2]) * (1.f / 3.f);
    const float p1 = e[3] * e[3] + e[4] * e[4] + e[5] * e[5];
    const float d0 = e[0] - q, d1 = e[1] - q, d2 = e[2] - q;
    const float p2 = d0 * d0 + d1 * d1 + d2 * d2 + 2.f * p1;
    float l1, l2, l3;
    if (p2 <= 0.f) {
        l1 = l2 = l3 = q;
    } else {
        const float p = sqrtf(p2 * (1.f / 6.f));
        const float ip = __fdividef(1.f, p);
        const float b0 = d0 * ip, b4 = d1 * ip, b8 = d2 * ip;
        const float b1 = e[3] * ip, b2 = e[4] * ip, b5 = e[5] * ip;
        const float detB = b0 * (b4 * b8 - b5 * b5) - b1 * (b1 * b8 - b5 * b2) + b2 * (b1 * b5 - b4 * b2);
        const float r = fminf(fmaxf(0.5f * detB, -1.f), 1.f);
        const float phi = acosf(r) * (1.f / 3.f);   // in [0, pi/3]
        // cos(phi + 2pi/3) = -cos(phi)/2 - sqrt(3)/2 sin(phi); MUFU sin/cos
        // (abs. error ~4e-7 on [0, pi/3]; e is scaled to unit max entry)
        float sp, cp;
        __sincosf(phi, &sp, &cp);
        l1 = q + 2.f * p * cp;
        l3 = q - p * (cp + 1.7320508075688772f * sp);
        l2 = 3.f * q - l1 - l3;
    }
    if (l3 >= 0.f) {
#pragma unroll
        for (int k = 0; k < 6; ++k) ep[k] = e[k];
        return;
    }
    if (l1 <= 0.f) {
#pragma unroll
        for (int k = 0; k < 6; ++k) ep[k] = 0.f;
        return;
    }
    const float e2[6] = {e[0] * e[0] + e[3] * e[3] + e[4] * e[4],
                         e[3] * e[3] + e[1] * e[1] + e[5] * e[5],
                         e[4] * e[4] + e[5] * e[5] + e[2] * e[2],
                         e[0] * e[3] + e[3] * e[1] + e[4] * e[5],
                         e[0] * e[4] + e[3] * e[5] + e[4] * e[2],
                         e[3] * e[4] + e[1] * e[5] + e[5] * e[2]};
    // isolated eigenvalue lk with projector (E - la I)(E - lb I) / ((lk-la)(lk-lb))
    const bool top = l2 <= 0.f;          // l1 alone positive: E+ = l1 P1
    const float lk = top ? l1 : l3, la = top ? l2 : l1, lb = top ? l3 : l2;
    const float c = __fdividef(lk, (lk - la) * (lk - lb));
    const float sab = la + lb, pab = la * lb;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const float pk = c * (e2[k] - sab * e[k] + (k < 3 ? pab : 0.f));
        ep[k] = top ? pk : e[k] - pk;
    }
}

// FP32 SVK + spectral split on symmetric storage (reference.py:94-116):
// E = (H + H^T + H^T H)/2, E+ by the closed form, S = s^2 S+ + S-
__device__ __forceinline__ void svk_split_f32(const float* H, float lam, float mu, float s, float* S,
                                              float& psi, float& psip) {
    // (r, c) of the symmetric components xx, yy, zz, xy, xz, yz
    constexpr int RR[6] = {0, 1, 2, 0, 0, 1}, CC[6] = {0, 1, 2, 1, 2, 2};
    float e[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const int r = RR[k], c = CC[k];
        e[k] = 0.5f * (H[3 * r + c] + H[3 * c + r] +
                       (H[r] * H[c] + H[3 + r] * H[3 + c] + H[6 + r] * H[6 + c]));
    }
    const float trE = e[0] + e[1] + e[2];
    const float trp = trE > 0.f ? trE : 0.f, trm = trE < 0.f ? trE : 0.f;
    // the split is positively homogeneous (E+(aE) = a E+(E)): run it on E
    // scaled to unit max entry so tiny strains far from the load do not
    // underflow (FTZ) into a 0/0 in the projector
    float m = 0.f;
#pragma unroll
    for (int k = 0; k < 6; ++k) m = fmaxf(m, fabsf(e[k]));
    float ep[6];
    if (m > 0.f) {
        const float im = __fdividef(1.f, m);
        float en[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) en[k] = e[k] * im;
        positive_part_sym(en, ep);
#pragma unroll
        for (int k = 0; k < 6; ++k) ep[k] *= m;
    } else {
#pragma unroll
        for (int k = 0; k < 6; ++k) ep[k] = 0.f;
    }
    const float s2 = s * s;
    float fp = 0.f, fm = 0.f, Ss[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const float a = ep[k], b = e[k] - ep[k];
        const float wgt = k < 3 ? 1.f : 2.f;     // off-diagonals count twice in E:E
        fp += wgt * a * a;
        fm += wgt * b * b;
        float sp = 2.f * mu * a, sm = 2.f * mu * b;
        if (k < 3) {
            sp += lam * trp;
            sm += lam * trm;
        }
        Ss[k] = s2 * sp + sm;
    }
    S[0] = Ss[0]; S[4] = Ss[1]; S[8] = Ss[2];
    S[1] = S[3] = Ss[3];
    S[2] = S[6] = Ss[4];
    S[5] = S[7] = Ss[5];
    const float pp = 0.5f * lam * trp * trp + mu * fp;
    const float pm = 0.5f * lam * trm * trm + mu * fm;
    psi = s2 * pp + pm;
    psip = pp;
}

// FP64 positive part E+ by the same closed form (trigonometric eigenvalues +
// the Sylvester projector of the sign-isolated eigenvalue), on full 3x3
// storage.  Its only ill-conditioned input is the isolated eigenvalue l_k
// when a same-sign partner lies within g of it: the trigonometric formula
// then carries an error ~ 2 eps p^2 / g (p = the deviatoric scale).  When
// g < TL_SPLIT_GAP * p that error could exceed ~1e-13 of |E|, and the split
// returns false: the caller runs the reference's cyclic Jacobi instead.
#define TL_SPLIT_GAP 1e-3
__device__ __forceinline__ bool positive_part64(const double* E, double* Ep) {
    const double q = (E[0] + E[4] + E[8]) * (1.0 / 3.0);
    const double o1 = E[1], o2 = E[2], o5 = E[5];
    const double d0 = E[0] - q, d1 = E[4] - q, d2 = E[8] - q;
    const double p2 = d0 * d0 + d1 * d1 + d2 * d2 + 2.0 * (o1 * o1 + o2 * o2 + o5 * o5);
    if (p2 <= 0.0) {   // E = q I
#pragma unroll
        for (int k = 0; k < 9; ++k) Ep[k] = q > 0.0 ? E[k] : 0.0;
        return true;
    }
    const double p = sqrt(p2 * (1.0 / 6.0));
    const double ip = 1.0 / p;
    const double b0 = d0 * ip, b4 = d1 * ip, b8 = d2 * ip;
    const double b1 = o1 * ip, b2 = o2 * ip, b5 = o5 * ip;
    const double detB = b0 * (b4 * b8 - b5 * b5) - b1 * (b1 * b8 - b5 * b2) + b2 * (b1 * b5 - b4 * b2);
    const double r = fmin(fmax(0.5 * detB, -1.0), 1.0);
    const double phi = acos(r) * (1.0 / 3.0);
    double sp, cp;
    sincos(phi, &sp, &cp);
    const double l1 = q + 2.0 * p * cp;
    const double l3 = q - p * (cp + 1.7320508075688772 * sp);
    const double l2 = 3.0 * q - l1 - l3;
    if (l3 >= 0.0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) Ep[k] = E[k];
        return true;
    }
    if (l1 <= 0.0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) Ep[k] = 0.0;
        return true;
    }
    const bool top = l2 <= 0.0;          // l1 alone positive: E+ = l1 P1
    const double lk = top ? l1 : l3, la = top ? l2 : l1, lb = top ? l3 : l2;
    if (fmin(fabs(lk - la), fabs(lk - lb)) < TL_SPLIT_GAP * p) return false;
    const double c = lk / ((lk - la) * (lk - lb));
    const double sab = la + lb, pab = la * lb;
#pragma unroll
    for (int rr = 0; rr < 3; ++rr)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            const double e2 = E[3 * rr] * E[cc] + E[3 * rr + 1] * E[3 + cc] + E[3 * rr + 2] * E[6 + cc];
            const double pk = c * (e2 - sab * E[3 * rr + cc] + (rr == cc ? pab : 0.0));
            Ep[3 * rr + cc] = top ? pk : E[3 * rr + cc] - pk;
        }
    return true;
}

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
    const R trp = trE > R(0) ? trE : R(0), trm = trE < R(0) ? trE : R(0);
    if (sizeof(R) == 4) {
        svk_split_f32(reinterpret_cast<const float*>(H), float(lam), float(mu), float(s),
                      reinterpret_cast<float*>(S), reinterpret_cast<float&>(psi),
                      reinterpret_cast<float&>(psip));
        return 0;
    }
    const R s2 = s * s;
    if constexpr (sizeof(R) == 8) {
        double Ep[9];
        if (positive_part64(E, Ep)) {
            double fp = 0.0, fm = 0.0;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const double a = Ep[k], m = E[k] - Ep[k];
                fp += a * a;
                fm += m * m;
                double sp = 2.0 * mu * a, sm = 2.0 * mu * m;
                if (k % 4 == 0) {
                    sp += lam * trp;
                    sm += lam * trm;
                }
                S[k] = s2 * sp + sm;
            }
            const double pp = 0.5 * lam * trp * trp + mu * fp;
            const double pm = 0.5 * lam * trm * trm + mu * fm;
            psi = s2 * pp + pm;
            psip = pp;
            return 0;
        }
    }
    R w[3], Q[9];
    const int sw = tl::eig3_jacobi(E, w, Q, jtol);
    R pp = R(0.5) * lam * trp * trp, pm = R(0.5) * lam * trm * trm;
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
// pair terms
// ---------------------------------------------------------------------------
template <typename R>
using V4 = typename tl::Vec4<R>::T;

// Kernel shape.  Both passes need fac_ij = (dW/dr)/r at r = |r0_ij|; it
// factors into a per-body constant times a shape w(r):
//   Wendland C2 : fac = -5 alpha/h^2 * t^3,          t = max(1 - r/(2h), 0)
//   cubic spline: fac = alpha/h * ((-3 + 2.25 q)/h   (q < 1)
//                                  | -0.75 (2-q)^2/r (1 <= q < 2) | 0)
// (kernel_geom.py:21-62 with q = r/h), so the pair loops carry w only and
// the constant (with V0 / m0 when uniform) is applied once per particle.
// r2 is floored so the self-padding entries of the neighbour slices (r0 = 0)
// give a finite w and vanishing terms.
template <typename R, int KIND>
__device__ __forceinline__ R kshape(R r2, R inv_h, R& rs) {
    rs = tl::rsqrt_floor(r2);
    const R r = r2 * rs;
    if (KIND == 2) {
        // neighbours lie inside the support (r < 2h, decided in FP64 at the
        // build), so t > 0; FP32 rounding near r = 2h can leave t ~ -1e-7,
        // whose t^3 ~ -1e-21 is below the mode's resolution -- the clamp is
        // kept only in FP64
        R t = R(1) - r * (R(0.5) * inv_h);
        if (sizeof(R) == 8) t = fmax(t, R(0));
        return t * t * t;
    }
    const R q = r * inv_h, tm = R(2) - q;
    return q < R(1) ? (R(-3) + R(2.25) * q) * inv_h : (q < R(2) ? R(-0.75) * tm * tm * rs : R(0));
}

template <typename R, int KIND>
__device__ __forceinline__ R kshape_const(const tl_body& b) {
    return KIND == 2 ? R(-5.0 * b.alpha * b.inv_h * b.inv_h) : R(b.alpha * b.inv_h);
}

// pass A pair (w = V0_j-weighted shape, wr = w r0):
//   D += (u_j - u_i) (x) wr ;  M += (s_i - s_j) / r^2  wr (x) r0
// (gated particles, s_i <= s_l, get F = I after the loop)
template <typename R, int DIM, bool FRAC, int KIND>
__device__ __forceinline__ void pair_a(R dx, R dy, R dz, const V4<R>& uj, R vj, bool uni,
                                       const V4<R>& ui, R inv_h, R* D, R* M) {
    const R r2 = dx * dx + dy * dy + dz * dz;
    R rs;
    R w = kshape<R, KIND>(r2, inv_h, rs);
    if (!uni) w *= vj;
    const R wx = w * dx, wz = w * dz;
    const R du0 = uj.x - ui.x, du2 = uj.z - ui.z;
    D[0] += du0 * wx; D[2] += du0 * wz;
    D[6] += du2 * wx; D[8] += du2 * wz;
    const R wy = DIM == 3 ? w * dy : R(0);
    if (DIM == 3) {
        const R du1 = uj.y - ui.y;
        D[1] += du0 * wy; D[7] += du2 * wy;
        D[3] += du1 * wx; D[4] += du1 * wy; D[5] += du1 * wz;
    }
    if (FRAC) {
        const R c = (ui.w - uj.w) * (rs * rs);
        const R cx = c * wx, cz = c * wz;
        M[0] += cx * dx; M[2] += cz * dz; M[4] += cx * dz;
        if (DIM == 3) {
            const R cy = c * wy;
            M[1] += cy * dy; M[3] += cx * dy; M[5] += cy * dz;
        }
    }
}

__device__ __forceinline__ float fdiv(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double fdiv(double a, double b) { return a / b; }

// pass B pair (w = m_j-weighted shape, wr = w r0):
//   s1 += wr ;  s2 += PL_j wr ;  s3 += (B2 G'^2 - B1 G') wr
// with G' = (v_i - v_j).r0 / (r^2 + 0.001 h^2); B2 = beta2 h^2, B1 = beta1 c0 h
template <typename R, int DIM, int KIND>
__device__ __forceinline__ void pair_b(R dx, R dy, R dz, const V4<R>& q0, const V4<R>& q1,
                                       const V4<R>& q2, R mj, bool uni, R vi0, R vi1, R vi2,
                                       bool visc, R inv_h, R eps_h2, R B2, R B1, R* s1, R* s2,
                                       R* s3) {
    const R r2 = dx * dx + dy * dy + dz * dz;
    R rs;
    R w = kshape<R, KIND>(r2, inv_h, rs);
    if (!uni) w *= mj;
    const R wx = w * dx, wz = w * dz;
    const R wy = DIM == 3 ? w * dy : R(0);
    s1[0] += wx; s1[2] += wz;
    // record layout (RecB): q0 = (PL00 PL10 PL01 PL11), q1 = (PL02 PL12 PL20 PL21),
    // q2 = (v0 v1 v2 PL22)
    if (DIM == 3) {
        s1[1] += wy;
        s2[0] = fma(q1.x, wz, fma(q0.z, wy, fma(q0.x, wx, s2[0])));
        s2[1] = fma(q1.y, wz, fma(q0.w, wy, fma(q0.y, wx, s2[1])));
        s2[2] = fma(q2.w, wz, fma(q1.w, wy, fma(q1.z, wx, s2[2])));
    } else {
        s2[0] = fma(q1.x, wz, fma(q0.x, wx, s2[0]));
        s2[2] = fma(q2.w, wz, fma(q1.z, wx, s2[2]));
    }
    if (visc) {
        const R dvr = (vi0 - q2.x) * dx + (DIM == 3 ? (vi1 - q2.y) * dy : R(0)) + (vi2 - q2.z) * dz;
        const R g = fdiv(dvr, r2 + eps_h2);
        const R pw = (B2 * g - B1) * g;
        s3[0] += pw * wx; s3[2] += pw * wz;
        if (DIM == 3) s3[1] += pw * wy;
    }
}

// explicit 32-bit shared-memory loads (slot byte offsets + per-CTA bases)
template <typename R>
__device__ __forceinline__ V4<R> lds4(uint32_t a);
template <>
__device__ __forceinline__ float4 lds4<float>(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a));
    return v;
}
template <>
__device__ __forceinline__ double4 lds4<double>(uint32_t a) {
    double4 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%4];\n\tld.shared.v2.f64 {%2, %3}, [%4+16];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "r"(a));
    return v;
}

// the 4 slot byte offsets of this lane's neighbour group k (staged in
// shared memory, or from global memory for oversized slot tables)
template <bool STAGED>
__device__ __forceinline__ uint2 slot_group(uint32_t sl_sh, const uint16_t* sl_g, int k) {
    if (STAGED) {
        uint2 v;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(sl_sh + 64u * k));
        return v;
    }
    return __ldg(reinterpret_cast<const uint2*>(sl_g + 32 * k));
}

// Visit this lane's len slots (raw slot values) group by group.  A warp's
// slices are padded to a multiple of 4; `len` is the warp's real longest
// row, so the last group runs only len % 4 pairs.  With the slot table in
// global memory (!STAGED: the tile's table did not fit next to its halo) the
// next group's load is issued before this group's pairs.
template <bool STAGED, typename F>
__device__ __forceinline__ void each_slot(uint32_t sl_sh, const uint16_t* sl_g, int len, F&& pair) {
    const int full = len & ~3;
    int k = 0;
    uint2 v = make_uint2(0u, 0u);
    if constexpr (STAGED) {
        for (; k < full; k += 4) {
            v = slot_group<true>(sl_sh, sl_g, k);
            pair(v.x & 0xffffu);
            pair(v.x >> 16);
            pair(v.y & 0xffffu);
            pair(v.y >> 16);
        }
        if (len & 3) v = slot_group<true>(sl_sh, sl_g, k);
    } else {
        if (len > 0) v = slot_group<false>(sl_sh, sl_g, 0);
        for (; k < full; k += 4) {
            const uint2 vn = k + 4 < len ? slot_group<false>(sl_sh, sl_g, k + 4) : v;
            pair(v.x & 0xffffu);
            pair(v.x >> 16);
            pair(v.y & 0xffffu);
            pair(v.y >> 16);
            v = vn;
        }
    }
    if (len & 3) {
        pair(v.x & 0xffffu);
        if ((len & 3) > 1) pair(v.x >> 16);
        if ((len & 3) > 2) pair(v.y & 0xffffu);
    }
}

// Neighbour loops over a staged tile.  Slots are slot * 16: the byte offset
// of the neighbour's FP32 position record (FP64 records are twice as wide);
// the gathered record sits at the same offset (pass A, one record) or
// three times it (pass B, three records).
// UNI (uniform V0 / m0) and STAGED (slot table in shared memory) are
// compile-time so the loop body has no per-pair predicates or branches.
template <typename R, int DIM, bool FRAC, int KIND, bool UNI, bool STAGED>
__device__ __forceinline__ void loop_a(uint32_t pos_sh, uint32_t rec_sh, uint32_t sl_sh,
                                       const uint16_t* sl_g, int len, const V4<R>& me,
                                       const V4<R>& ui, R inv_h, R* D, R* M) {
    constexpr uint32_t U = sizeof(V4<R>) / 16;   // 16-byte units per record
    auto pair = [&](uint32_t o) {
        const V4<R> pj = lds4<R>(pos_sh + o);
        const V4<R> uj = lds4<R>(rec_sh + o);
        pair_a<R, DIM, FRAC, KIND>(me.x - pj.x, DIM == 3 ? me.y - pj.y : R(0), me.z - pj.z, uj, pj.w,
                                   UNI, ui, inv_h, D, M);
    };
    each_slot<STAGED>(sl_sh, sl_g, len, [&](uint32_t sl) { pair(U * sl); });
}

template <typename R, int DIM, int KIND, bool UNI, bool STAGED, bool VISC>
__device__ __forceinline__ void loop_b(uint32_t pos_sh, uint32_t rec_sh, uint32_t sl_sh,
                                       const uint16_t* sl_g, int len, const V4<R>& me, R vi0, R vi1,
                                       R vi2, R inv_h, R eps_h2, R B2, R B1, R* s1, R* s2, R* s3) {
    constexpr uint32_t U = sizeof(V4<R>) / 16;
    auto pair = [&](uint32_t o) {
        const V4<R> pj = lds4<R>(pos_sh + o);
        const uint32_t ra = rec_sh + 3u * o;
        pair_b<R, DIM, KIND>(me.x - pj.x, DIM == 3 ? me.y - pj.y : R(0), me.z - pj.z, lds4<R>(ra),
                             lds4<R>(ra + sizeof(V4<R>)), lds4<R>(ra + 2 * sizeof(V4<R>)), pj.w, UNI,
                             vi0, vi1, vi2, VISC, inv_h, eps_h2, B2, B1, s1, s2, s3);
    };
    each_slot<STAGED>(sl_sh, sl_g, len, [&](uint32_t sl) { pair(U * sl); });
}

// FP32 3D pass-A loop on packed FP32x2 arithmetic (Blackwell FFMA2 / FADD2 /
// FMUL2, a scalar operand broadcast for free): the same pair terms as
// pair_a, about a quarter fewer issued instructions per pair.  It works on
// d' = x_j - x_i = -r0 (one packed subtract with -x_i precomputed), so the
// D it returns is negated; M is even in r0.
struct AccA2 {
    float2 D01, D34, D67, D25;   // (D0,D1) (D3,D4) (D6,D7) (D2,D5)
    float D8;
    float2 M01;                  // (xx, yy)
    float M2, M3, M4, M5;        // zz, xy, xz, yz
};

template <bool FRAC, int KIND, bool UNI>
__device__ __forceinline__ void pair_a_f2(const float4& pj, const float4& uj, const float2 nme_xy,
                                          float nme_z, const float2 nui_xy, float nui_z, float ui_s,
                                          float inv_h, AccA2& a) {
    const float2 dxy = __fadd2_rn(make_float2(pj.x, pj.y), nme_xy);   // -(r0.x, r0.y)
    const float dz = pj.z + nme_z;
    const float r2 = fmaf(dz, dz, fmaf(dxy.y, dxy.y, dxy.x * dxy.x));
    float rs;
    float w = kshape<float, KIND>(r2, inv_h, rs);
    if (!UNI) w *= pj.w;
    const float2 wxy = __fmul2_rn(make_float2(w, w), dxy);
    const float wz = w * dz;
    const float2 du01 = __fadd2_rn(make_float2(uj.x, uj.y), nui_xy);
    const float du2 = uj.z + nui_z;
    a.D01 = __ffma2_rn(make_float2(du01.x, du01.x), wxy, a.D01);
    a.D34 = __ffma2_rn(make_float2(du01.y, du01.y), wxy, a.D34);
    a.D67 = __ffma2_rn(make_float2(du2, du2), wxy, a.D67);
    a.D25 = __ffma2_rn(du01, make_float2(wz, wz), a.D25);
    a.D8 = fmaf(du2, wz, a.D8);
    if (FRAC) {
        const float c = (ui_s - uj.w) * (rs * rs);
        const float2 cxy = __fmul2_rn(make_float2(c, c), wxy);
        const float cz = c * wz;
        a.M01 = __ffma2_rn(cxy, dxy, a.M01);
        a.M2 = fmaf(cz, dz, a.M2);
        a.M3 = fmaf(cxy.x, dxy.y, a.M3);
        a.M4 = fmaf(cxy.x, dz, a.M4);
        a.M5 = fmaf(cxy.y, dz, a.M5);
    }
}

template <bool FRAC, int KIND, bool UNI, bool STAGED>
__device__ __forceinline__ void loop_a_f2(uint32_t pos_sh, uint32_t rec_sh, uint32_t sl_sh,
                                          const uint16_t* sl_g, int len, const float4& me,
                                          const float4& ui, float inv_h, float* D, float* M) {
    AccA2 a;
    a.D01 = a.D34 = a.D67 = a.D25 = a.M01 = make_float2(0.f, 0.f);
    a.D8 = a.M2 = a.M3 = a.M4 = a.M5 = 0.f;
    const float2 nme = make_float2(-me.x, -me.y), nui = make_float2(-ui.x, -ui.y);
    const float nmz = -me.z, nuz = -ui.z;
    auto pair = [&](uint32_t o) {
        pair_a_f2<FRAC, KIND, UNI>(lds4<float>(pos_sh + o), lds4<float>(rec_sh + o), nme, nmz, nui,
                                   nuz, ui.w, inv_h, a);
    };
    each_slot<STAGED>(sl_sh, sl_g, len, pair);
    // back to row-major D (= -D') and the (xx yy zz xy xz yz) M of pair_a
    D[0] = -a.D01.x; D[1] = -a.D01.y; D[2] = -a.D25.x;
    D[3] = -a.D34.x; D[4] = -a.D34.y; D[5] = -a.D25.y;
    D[6] = -a.D67.x; D[7] = -a.D67.y; D[8] = -a.D8;
    M[0] = a.M01.x; M[1] = a.M01.y; M[2] = a.M2; M[3] = a.M3; M[4] = a.M4; M[5] = a.M5;
}

// ---------------------------------------------------------------------------
// bond-class pair loops (b.ncls > 0, FP32): slot entry e = (class << 10) |
// slot.  The pair geometry comes from the class table -- W = w(r) r0,
// kappa = 1/(w (r^2 + eps h^2)), U = r0/r^2, computed once per body in FP64
// from the lattice separation (kernel_geom.StepLayout.bond_classes) --
// instead of a staged position record: no position load, no r, rsqrt or
// kernel shape per pair.  A warp's lanes mostly share a class at a given k
// (Morton bricks of one lattice), so the table loads are broadcasts.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t geo_slot(uint32_t e) { return e & 1023u; }
__device__ __forceinline__ uint32_t geo_cls(uint32_t e) { return (e >> 10) * 32u; }
__device__ __forceinline__ uint32_t geo_cls64(uint32_t e) { return (e >> 10) * 64u; }

// The tiled passes' bond-class entries as kernel parameters: read through
// the constant cache (a broadcast where a warp's lanes share the class, which
// a lattice interior's CSR-ordered rows do) instead of shared-memory loads on
// the record loads' pipe.  Pass B needs (W, kappa), pass A also U.
#define TL_TILE_MAX_CLASSES 64
template <typename R>
struct ClsTab {
    V4<R> W[TL_TILE_MAX_CLASSES];
};
template <typename R>
struct ClsTabA {
    V4<R> W[TL_TILE_MAX_CLASSES];
    V4<R> U[TL_TILE_MAX_CLASSES];
};

// pass A, FP32 3D, packed FP32x2: D += (u_j - u_i) (x) W ; M += (s_i - s_j) W (x) U
template <bool FRAC, bool STAGED, bool CC = false>
__device__ __forceinline__ void loop_a_geo_f2(uint32_t rec_sh, uint32_t cls_sh, uint32_t sl_sh,
                                              const uint16_t* sl_g, int len, const float4& ui,
                                              float* D, float* M,
                                              const ClsTabA<float>* ct = nullptr) {
    float2 D01 = make_float2(0.f, 0.f), D34 = D01, D67 = D01, D25 = D01, M01 = D01;
    float D8 = 0.f, M2 = 0.f, M3 = 0.f, M4 = 0.f, M5 = 0.f;
    const float2 nui = make_float2(-ui.x, -ui.y);
    const float nuz = -ui.z;
    each_slot<STAGED>(sl_sh, sl_g, len, [&](uint32_t e) {
        const uint32_t c = cls_sh + geo_cls(e);
        const float4 W = CC ? ct->W[e >> 10] : lds4<float>(c);
        const float4 uj = lds4<float>(rec_sh + 16u * geo_slot(e));
        const float2 wxy = make_float2(W.x, W.y);
        const float2 du01 = __fadd2_rn(make_float2(uj.x, uj.y), nui);
        const float du2 = uj.z + nuz;
        D01 = __ffma2_rn(make_float2(du01.x, du01.x), wxy, D01);
        D34 = __ffma2_rn(make_float2(du01.y, du01.y), wxy, D34);
        D67 = __ffma2_rn(make_float2(du2, du2), wxy, D67);
        D25 = __ffma2_rn(du01, make_float2(W.z, W.z), D25);
        D8 = fmaf(du2, W.z, D8);
        if (FRAC) {
            const float4 U = CC ? ct->U[e >> 10] : lds4<float>(c + 16u);
            const float ds = ui.w - uj.w;
            const float2 cw = __fmul2_rn(make_float2(ds, ds), wxy);
            const float cz = ds * W.z;
            M01 = __ffma2_rn(cw, make_float2(U.x, U.y), M01);
            M2 = fmaf(cz, U.z, M2);
            M3 = fmaf(cw.x, U.y, M3);
            M4 = fmaf(cw.x, U.z, M4);
            M5 = fmaf(cw.y, U.z, M5);
        }
    });
    D[0] = D01.x; D[1] = D01.y; D[2] = D25.x;
    D[3] = D34.x; D[4] = D34.y; D[5] = D25.y;
    D[6] = D67.x; D[7] = D67.y; D[8] = D8;
    M[0] = M01.x; M[1] = M01.y; M[2] = M2; M[3] = M3; M[4] = M4; M[5] = M5;
}

// pass A, FP32 2D (x-z plane): the scalar form of the same terms
template <bool FRAC, bool STAGED, bool CC = false>
__device__ __forceinline__ void loop_a_geo_2d(uint32_t rec_sh, uint32_t cls_sh, uint32_t sl_sh,
                                              const uint16_t* sl_g, int len, const float4& ui,
                                              float* D, float* M,
                                              const ClsTabA<float>* ct = nullptr) {
    each_slot<STAGED>(sl_sh, sl_g, len, [&](uint32_t e) {
        const uint32_t c = cls_sh + geo_cls(e);
        const float4 W = CC ? ct->W[e >> 10] : lds4<float>(c);
        const float4 uj = lds4<float>(rec_sh + 16u * geo_slot(e));
        const float du0 = uj.x - ui.x, du2 = uj.z - ui.z;
        D[0] = fmaf(du0, W.x, D[0]); D[2] = fmaf(du0, W.z, D[2]);
        D[6] = fmaf(du2, W.x, D[6]); D[8] = fmaf(du2, W.z, D[8]);
        if (FRAC) {
            const float4 U = CC ? ct->U[e >> 10] : lds4<float>(c + 16u);
            const float ds = ui.w - uj.w;
            const float cx = ds * W.x, cz = ds * W.z;
            M[0] = fmaf(cx, U.x, M[0]); M[2] = fmaf(cz, U.z, M[2]); M[4] = fmaf(cx, U.z, M[4]);
        }
    });
}

// pass B: s1 += W ; s2 += PL_j W ; s3 += (B2 g^2 - B1 g) W with
// g = (v_i - v_j).W kappa = (v_i - v_j).r0 / (r^2 + eps h^2).  3D runs on
// packed FP32x2: the RecB layout pairs rows 0 and 1 of PL_j column by column,
// so (s2_0, s2_1) takes three FFMA2 with a broadcast W component, and
// (s1_0, s1_1), (s3_0, s3_1) and (v_i - v_j)_{0,1} are register pairs too.
// CC: (W, kappa) from the ClsTab kernel parameter, else from shared memory
template <int DIM, bool STAGED, bool VISC, bool CC = false>
__device__ __forceinline__ void loop_b_geo(uint32_t rec_sh, uint32_t cls_sh, uint32_t sl_sh,
                                           const uint16_t* sl_g, int len, float vi0, float vi1,
                                           float vi2, float B2, float B1, float* s1, float* s2,
                                           float* s3, const ClsTab<float>* ct = nullptr) {
    if constexpr (DIM == 3) {
        float2 s1a = make_float2(0.f, 0.f), s2a = s1a, s3a = s1a;
        float s1b = 0.f, s2b = 0.f, s3b = 0.f;
        const float2 vi01 = make_float2(vi0, vi1);
        const float2 neg1 = make_float2(-1.f, -1.f);
        each_slot<STAGED>(sl_sh, sl_g, len, [&](uint32_t e) {
            const float4 W = CC ? ct->W[e >> 10] : lds4<float>(cls_sh + geo_cls(e));
            const uint32_t ra = rec_sh + 48u * geo_slot(e);
            const float4 q0 = lds4<float>(ra), q1 = lds4<float>(ra + 16u), q2 = lds4<float>(ra + 32u);
            const float2 wxy = make_float2(W.x, W.y);
            s1a = __fadd2_rn(s1a, wxy);
            s1b += W.z;
            s2a = __ffma2_rn(make_float2(q0.x, q0.y), make_float2(W.x, W.x), s2a);
            s2a = __ffma2_rn(make_float2(q0.z, q0.w), make_float2(W.y, W.y), s2a);
            s2a = __ffma2_rn(make_float2(q1.x, q1.y), make_float2(W.z, W.z), s2a);
            s2b = fmaf(q2.w, W.z, fmaf(q1.w, W.y, fmaf(q1.z, W.x, s2b)));
            if (VISC) {
                const float2 dv = __ffma2_rn(make_float2(q2.x, q2.y), neg1, vi01);
                const float2 pr = __fmul2_rn(dv, wxy);
                const float dvw = fmaf(vi2 - q2.z, W.z, pr.x + pr.y);
                const float g = dvw * W.w;
                const float pw = (B2 * g - B1) * g;
                s3a = __ffma2_rn(make_float2(pw, pw), wxy, s3a);
                s3b = fmaf(pw, W.z, s3b);
            }
        });
        s1[0] = s1a.x; s1[1] = s1a.y; s1[2] = s1b;
        s2[0] = s2a.x; s2[1] = s2a.y; s2[2] = s2b;
        s3[0] = s3a.x; s3[1] = s3a.y; s3[2] = s3b;
    } else {
        each_slot<STAGED>(sl_sh, sl_g, len, [&](uint32_t e) {
            const float4 W = CC ? ct->W[e >> 10] : lds4<float>(cls_sh + geo_cls(e));
            const uint32_t ra = rec_sh + 48u * geo_slot(e);
            const float4 q0 = lds4<float>(ra), q1 = lds4<float>(ra + 16u), q2 = lds4<float>(ra + 32u);
            s1[0] += W.x; s1[2] += W.z;
            s2[0] = fmaf(q1.x, W.z, fmaf(q0.x, W.x, s2[0]));
            s2[2] = fmaf(q2.w, W.z, fmaf(q1.z, W.x, s2[2]));
            if (VISC) {
                const float dvw = (vi0 - q2.x) * W.x + (vi2 - q2.z) * W.z;
                const float g = dvw * W.w;
                const float pw = (B2 * g - B1) * g;
                s3[0] = fmaf(pw, W.x, s3[0]); s3[2] = fmaf(pw, W.z, s3[2]);
            }
        });
    }
}

// FP64 bond-class loops (scalar): the same pair terms as pair_a / pair_b with
// the class table's W, kappa, U in place of the per-pair geometry
template <int DIM, bool FRAC, bool STAGED>
__device__ __forceinline__ void loop_a_geo64(uint32_t rec_sh, uint32_t cls_sh, uint32_t sl_sh,
                                             const uint16_t* sl_g, int len, const double4& ui,
                                             double* D, double* M) {
    each_slot<STAGED>(sl_sh, sl_g, len, [&](uint32_t e) {
        const uint32_t c = cls_sh + geo_cls64(e);
        const double4 W = lds4<double>(c);
        const double4 uj = lds4<double>(rec_sh + 32u * geo_slot(e));
        const double du0 = uj.x - ui.x, du2 = uj.z - ui.z;
        D[0] = fma(du0, W.x, D[0]); D[2] = fma(du0, W.z, D[2]);
        D[6] = fma(du2, W.x, D[6]); D[8] = fma(du2, W.z, D[8]);
        if (DIM == 3) {
            const double du1 = uj.y - ui.y;
            D[1] = fma(du0, W.y, D[1]); D[7] = fma(du2, W.y, D[7]);
            D[3] = fma(du1, W.x, D[3]); D[4] = fma(du1, W.y, D[4]); D[5] = fma(du1, W.z, D[5]);
        }
        if (FRAC) {
            const double4 U = lds4<double>(c + 32u);
            const double ds = ui.w - uj.w;
            const double cx = ds * W.x, cz = ds * W.z;
            M[0] = fma(cx, U.x, M[0]); M[2] = fma(cz, U.z, M[2]); M[4] = fma(cx, U.z, M[4]);
            if (DIM == 3) {
                const double cy = ds * W.y;
                M[1] = fma(cy, U.y, M[1]); M[3] = fma(cx, U.y, M[3]); M[5] = fma(cy, U.z, M[5]);
            }
        }
    });
}

template <int DIM, bool STAGED, bool VISC, bool CC = false>
__device__ __forceinline__ void loop_b_geo64(uint32_t rec_sh, uint32_t cls_sh, uint32_t sl_sh,
                                             const uint16_t* sl_g, int len, double vi0, double vi1,
                                             double vi2, double B2, double B1, double* s1,
                                             double* s2, double* s3,
                                             const ClsTab<double>* ct = nullptr) {
    each_slot<STAGED>(sl_sh, sl_g, len, [&](uint32_t e) {
        const double4 W = CC ? ct->W[e >> 10] : lds4<double>(cls_sh + geo_cls64(e));
        const uint32_t ra = rec_sh + 96u * geo_slot(e);
        const double4 q0 = lds4<double>(ra), q1 = lds4<double>(ra + 32u), q2 = lds4<double>(ra + 64u);
        s1[0] += W.x; s1[2] += W.z;
        if (DIM == 3) {
            s1[1] += W.y;
            s2[0] = fma(q1.x, W.z, fma(q0.z, W.y, fma(q0.x, W.x, s2[0])));
            s2[1] = fma(q1.y, W.z, fma(q0.w, W.y, fma(q0.y, W.x, s2[1])));
            s2[2] = fma(q2.w, W.z, fma(q1.w, W.y, fma(q1.z, W.x, s2[2])));
        } else {
            s2[0] = fma(q1.x, W.z, fma(q0.x, W.x, s2[0]));
            s2[2] = fma(q2.w, W.z, fma(q1.z, W.x, s2[2]));
        }
        if (VISC) {
            const double dvw = (vi0 - q2.x) * W.x + (DIM == 3 ? (vi1 - q2.y) * W.y : 0.0) +
                               (vi2 - q2.z) * W.z;
            const double g = dvw * W.w;
            const double pw = (B2 * g - B1) * g;
            s3[0] = fma(pw, W.x, s3[0]); s3[2] = fma(pw, W.z, s3[2]);
            if (DIM == 3) s3[1] = fma(pw, W.y, s3[1]);
        }
    });
}

// Shared-memory tile of a CTA.  Two arrays indexed by slot, then the CTA's
// block of the neighbour-slot table:
//   pos[slot]             the staged position record (x, y, z, w) -- a copy of
//                         the tile's block of tl_tile_pos records;
//   rec[slot * NREC + r]  the NREC gathered records of the particle, stored
//                         contiguously (48-byte FP32 pass-B records: the
//                         stride 3 is odd, so slots distinct mod 8 still hit
//                         distinct bank groups).
// Members sit at slot p - p0, halo particles at their residue-aligned hslot
// (tiles.cu k_hslots).  The capacity S = tile + hmax is the same for every
// CTA of a launch.
//
// Bond-class mode (b.ncls > 0; FP32 lattice bodies with uniform V0, m0):
// no position records at all.  The pair geometry is a per-class table entry
// (tl_body.bcls) selected by the class field of the slot entry, staged after
// the slot block:
//   rec[slot * NREC + r] | slots | cls[2 * class + {0, 1}] = (W, kappa), (U, 0)
template <typename R, int NREC>
struct Tile {
    V4<R>* pos;        // nullptr in bond-class mode
    V4<R>* rec;
    uint16_t* slots;   // the CTA's block of the slot table (its warps' slices)
    V4<R>* cls;        // bond-class table (bond-class mode)
};

__host__ __device__ constexpr size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

template <typename R, int NREC>
__host__ __device__ constexpr size_t tile_bytes(int S, int slmax, int ncls = 0) {
    return ncls > 0 ? (size_t)S * NREC * sizeof(V4<R>) + align16((size_t)slmax * sizeof(uint16_t)) +
                          (size_t)ncls * 2 * sizeof(V4<R>)
                    : (size_t)S * (NREC + 1) * sizeof(V4<R>) + (size_t)slmax * sizeof(uint16_t);
}

template <typename R, int NREC>
__device__ __forceinline__ Tile<R, NREC> tile_layout(unsigned char* smem, int S, int slmax = 0,
                                                     int ncls = 0) {
    Tile<R, NREC> t;
    if (ncls > 0) {
        t.pos = nullptr;
        t.rec = reinterpret_cast<V4<R>*>(smem);
        t.slots = reinterpret_cast<uint16_t*>(t.rec + (size_t)S * NREC);
        t.cls = reinterpret_cast<V4<R>*>(reinterpret_cast<unsigned char*>(t.slots) +
                                          align16((size_t)slmax * sizeof(uint16_t)));
        return t;
    }
    t.pos = reinterpret_cast<V4<R>*>(smem);
    t.rec = t.pos + S;
    t.slots = reinterpret_cast<uint16_t*>(t.rec + (size_t)S * NREC);
    t.cls = nullptr;
    return t;
}

// Stage a tile with asynchronous copies only: thread 0 arms the barrier and
// issues three TMA bulk copies (the contiguous position block, the members'
// records, the CTA's neighbour-slot block); every thread then issues 16-byte
// LDGSTS gathers of the halo records.  No register round trip, every load of
// the CTA in flight at once.
template <typename R, int NREC>
__device__ __forceinline__ void stage_tile(const tl_body& b, const Tile<R, NREC>& t, int64_t tile,
                                           const void* tpos, const R* src, uint64_t* bar) {
    const int T = b.tile;
    const int64_t p0 = tile * T;
    const int64_t hb = b.hoff[tile];
    const int H = (int)(b.hoff[tile + 1] - hb);
    if (threadIdx.x == 0) {
        const int64_t nmem = min((int64_t)T, b.n - p0);
        const int64_t r0 = t.pos ? b.toff[tile] : 0;
        const uint32_t pos_bytes =
            t.pos ? (uint32_t)((b.toff[tile + 1] - r0) * sizeof(V4<R>)) : 0u;
        const uint32_t mem_bytes = (uint32_t)(nmem * NREC * sizeof(V4<R>));
        const int64_t w0 = p0 >> 5, w1 = min(w0 + T / 32, (b.n + 31) >> 5);
        const uint32_t sl_bytes =
            b.slmax > 0 ? (uint32_t)((b.soff[w1] - b.soff[w0]) * sizeof(uint16_t)) : 0u;
        const uint32_t cls_bytes = t.cls ? (uint32_t)(b.ncls * 2 * sizeof(V4<R>)) : 0u;
        tl::mbar_init(bar, 1);
        tl::mbar_expect_tx(bar, pos_bytes + mem_bytes + sl_bytes + cls_bytes);
        if (pos_bytes) tl::bulk_g2s(t.pos, static_cast<const V4<R>*>(tpos) + r0, pos_bytes, bar);
        tl::bulk_g2s(t.rec, src + p0 * 4 * NREC, mem_bytes, bar);
        if (sl_bytes) tl::bulk_g2s(t.slots, b.slots + b.soff[w0], sl_bytes, bar);
        if (cls_bytes) tl::bulk_g2s(t.cls, static_cast<const V4<R>*>(b.bcls), cls_bytes, bar);
    }
    constexpr int CH = (int)(sizeof(V4<R>) / 16);   // 16-byte chunks per record
    for (int s = threadIdx.x; s < H; s += blockDim.x) {
        const int64_t q = b.halo[hb + s];
        const int d = b.hslot[hb + s];
        const char* g = reinterpret_cast<const char*>(src + q * 4 * NREC);
        char* sm = reinterpret_cast<char*>(t.rec + (int64_t)d * NREC);
#pragma unroll
        for (int c = 0; c < NREC * CH; ++c) tl::cp_async16(sm + 16 * c, g + 16 * c);
    }
    tl::cp_async_wait_all();
    __syncthreads();
    tl::mbar_wait(bar, 0);
}

// Tile of this CTA.  Multi-GPU slabs launch a tiled pass in two parts -- the
// tiles that read no halo rows while the halo exchange is in flight, then
// the rest -- through the tile list tlist[tbase + blockIdx.x].
__device__ __forceinline__ int64_t tile_of(const tl_body& b, bool tiled) {
    return (tiled && b.tlist) ? (int64_t)b.tlist[b.tbase + blockIdx.x] : (int64_t)blockIdx.x;
}

// L2 prefetch of the tile's own-particle planes the epilogue reads after the
// neighbour loop, issued by one thread while the tile is being staged
template <typename T>
__device__ __forceinline__ void prefetch_planes(const void* base, int64_t stride, int nplanes,
                                                int64_t p0, int64_t cnt) {
    if (!base) return;
    const T* p = static_cast<const T*>(base);
    for (int c = 0; c < nplanes; ++c) tl::l2_prefetch(p + c * stride + p0, cnt * sizeof(T));
}

template <typename R, int MODEL, bool FRAC>
__device__ __forceinline__ void prefetch_own_a(const tl_body& b, int64_t p0) {
    const int64_t cnt = min((int64_t)b.tile, b.n - p0), N = b.n_all;
    prefetch_planes<R>(b.L, N, 9, p0, cnt);
    prefetch_planes<R>(b.v, N, 3, p0, cnt);
    if (FRAC) {
        prefetch_planes<R>(b.sdot, N, 1, p0, cnt);
        prefetch_planes<R>(b.Hh, N, 1, p0, cnt);
    }
    if (MODEL == 3) {
        prefetch_planes<R>(b.Cpd, N, 6, p0, cnt);
        prefetch_planes<R>(b.epbar, N, 1, p0, cnt);
    }
}

template <typename R, bool FRAC>
__device__ __forceinline__ void prefetch_own_b(const tl_body& b, int64_t p0) {
    const int64_t cnt = min((int64_t)b.tile, b.n - p0), N = b.n_all;
    if (b.visc) prefetch_planes<R>(b.al, N, 9, p0, cnt);
    tl::l2_prefetch(static_cast<const R*>(b.us) + 4 * p0, cnt * 4 * sizeof(R));
    if (FRAC) {
        prefetch_planes<R>(b.sdot, N, 1, p0, cnt);
        prefetch_planes<R>(b.sddot, N, 1, p0, cnt);
    }
    if (b.bcmask) prefetch_planes<int32_t>(b.bcmask, N, 1, p0, cnt);
}

// ---------------------------------------------------------------------------
// pass A
// ---------------------------------------------------------------------------
// Pass A after the neighbour sums, shared by the tiled, L2-gather and brick
// kernels: D = sum (u_j - u_i) (x) w r0 and M = sum (s_i - s_j) w r0 r0^T / r^2
// (without the kernel constant) in, then F, the constitutive update, the phase
// field, P L_i, the viscosity tensor and the pass-B record of particle i.
// Returns this particle's plastic work increment dwp V0 (J2).
template <typename R, int DIM, int MODEL, bool FRAC, int KIND>
__device__ __forceinline__ double a_finish(const tl_body& b, int64_t i, R* D, R* M, R si,
                                          bool gated) {
    const int64_t N = b.n_all;
    const bool uni = b.uniform != 0;
    double pw = 0.0;
    {   // kernel constant (and V0 when uniform), once per particle
        const R ck = kshape_const<R, KIND>(b) * (uni ? R(b.V0c) : R(1));
#pragma unroll
        for (int q = 0; q < 9; ++q) D[q] *= ck;
#pragma unroll
        for (int q = 0; q < 6; ++q) M[q] *= R(2) * ck;
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
        if (nonspd) {
            // the reference raises here (constitutive.py:191-194): no stress,
            // no plastic update for this particle; pass B will not run
#pragma unroll
            for (int q = 0; q < 9; ++q) Sd[q] = 0.0;
            psid = dwp = 0.0;
            atomicMin((long long*)&b.counters[2], (long long)(b.perm ? b.perm[i] : i));
            flag_step_error(b.clock, 1);
        }
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
        // fracture.py:25-32 with the divisions as host-side reciprocals
        const R eps0 = R(b.eps0), c0 = R(b.c0), ieps = R(b.inv_eps0);
        const R ratio = Hn * R(b.inv_Gc);
        const R damp = R(2) * sqrt(R(4) * eps0 * ratio + R(1)) * R(b.inv_c0);
        const R sd = static_cast<const R*>(b.sdot)[i];
        static_cast<R*>(b.sddot)[i] =
            (R(0.5) * c0 * c0 * ieps) *
            (R(2) * eps0 * lap + R(0.5) * (R(1) - si) * ieps - damp * sd - R(2) * si * ratio);
    }
    if (b.Fh) {   // F for the opt-in hourglass control (tl_hourglass)
        R* Fh = static_cast<R*>(b.Fh);
#pragma unroll
        for (int q = 0; q < 9; ++q) Fh[q * N + i] = Hm[q] + ((q % 4 == 0) ? R(1) : R(0));
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
    // RecB layout: rows 0 and 1 of PL interleaved by column (packed FP32x2
    // sums in pass B), then row 2, v, PL22
    tl::st4(rb, PL[0], PL[3], PL[1], PL[4]);
    tl::st4(rb + 4, PL[2], PL[5], PL[6], PL[7]);
    tl::st4(rb + 8, vv[i], vv[N + i], vv[2 * N + i], PL[8]);
    if (b.peer_slot) {   // the record into the neighbouring ranks' halo rows (NVLink)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int32_t slot = b.peer_slot[k * N + i];
            if (slot >= 0) {
                R* pr = static_cast<R*>(b.peer_rb[k]) + 12 * (int64_t)slot;
                tl::st4(pr, PL[0], PL[3], PL[1], PL[4]);
                tl::st4(pr + 4, PL[2], PL[5], PL[6], PL[7]);
                tl::st4(pr + 8, vv[i], vv[N + i], vv[2 * N + i], PL[8]);
            }
        }
    }
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
        if (noconv) {
            atomicAdd((unsigned long long*)&b.counters[1], 1ull);
            flag_step_error(b.clock, 1);
        }
    }
    return pw;
}

template <typename R, int DIM, int MODEL, bool FRAC, int KIND, int G, bool TILED>
__global__ void __launch_bounds__(kThreads, TL_MINB_A(R, TILED))
    k_pass_a(const __grid_constant__ tl_body b, const __grid_constant__ ClsTabA<R> ct) {
    extern __shared__ __align__(16) unsigned char smem[];
    tl::pdl_enter();
    // a CTA of blockDim.x threads owns blockDim.x consecutive particles (TILED:
    // one shared tile of b.tile == blockDim.x particles); one particle per
    // thread -- larger tiles looped over by 256 threads measured slower
    // (shared memory per CTA cuts residency)
    const int64_t tb = tile_of(b, TILED);
    const int64_t p0 = tb * (int64_t)blockDim.x;
    __shared__ double s_pw[kThreads / 32];
    double pw = 0.0;
    if (halted(b)) return;
    const R* us = static_cast<const R*>(b.us);
    const bool uni = b.uniform != 0;
    // tile staging (TILED): every thread of the CTA takes part
    Tile<R, 1> tl_;
    __shared__ uint64_t bar;
    if (TILED) {
        if (threadIdx.x == 32) prefetch_own_a<R, MODEL, FRAC>(b, p0);
        tl_ = tile_layout<R, 1>(smem, b.tile + b.hmax, b.slmax, b.ncls);
        stage_tile<R, 1>(b, tl_, tb, b.tpos_a, us, &bar);
    }
    const int ms = (int)threadIdx.x;   // member slot
    const int64_t i = p0 + ms;
    if (i < b.n) {
        const int64_t N = b.n_all;
        const int lane = (int)(i & 31);
        const int64_t w = i >> 5;
        const int64_t base = b.soff[w];
        const int len = (int)((b.soff[w + 1] - base) >> 5);
        const auto ui = TILED ? tl_.rec[ms] : tl::ld4(us + 4 * i);
        const R si = ui.w;
        const bool gated = FRAC && si <= R(b.s_l);
        const R inv_h = R(b.inv_h);
        R D[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) D[q] = R(0);
        R M[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};   // xx yy zz xy xz yz
        if (TILED && tl_.cls != nullptr) {
          // bond classes: geometry from the class table, no positions
          const uint32_t rec_sh = tl::smem_u32(tl_.rec), cls_sh = tl::smem_u32(tl_.cls);
          const uint32_t sl_sh = tl::smem_u32(tl_.slots + (base - b.soff[p0 >> 5]) + lane * G);
          const uint16_t* slg = b.slots + base + lane * G;
          const int lenr = b.wlen ? (int)b.wlen[w] : len;
          if constexpr (sizeof(R) == 8) {
            const double4& uid = reinterpret_cast<const double4&>(ui);
            double* Dd = reinterpret_cast<double*>(D);
            double* Md = reinterpret_cast<double*>(M);
            if (b.slmax > 0) loop_a_geo64<DIM, FRAC, true>(rec_sh, cls_sh, sl_sh, slg, lenr, uid, Dd, Md);
            else loop_a_geo64<DIM, FRAC, false>(rec_sh, cls_sh, sl_sh, slg, lenr, uid, Dd, Md);
          } else {
            const float4& uif = reinterpret_cast<const float4&>(ui);
            float* Df = reinterpret_cast<float*>(D);
            float* Mf = reinterpret_cast<float*>(M);
            if constexpr (DIM == 3) {
                // 3D keeps the shared-memory table: the constant-bank one measured
                // flat here and the extra loop variant cost pass A 0.7 % (C4)
                if (b.slmax > 0) loop_a_geo_f2<FRAC, true>(rec_sh, cls_sh, sl_sh, slg, lenr, uif, Df, Mf);
                else loop_a_geo_f2<FRAC, false>(rec_sh, cls_sh, sl_sh, slg, lenr, uif, Df, Mf);
            } else {
                if (b.bcls_host && b.slmax > 0)
                    loop_a_geo_2d<FRAC, true, true>(rec_sh, cls_sh, sl_sh, slg, lenr, uif, Df, Mf, &ct);
                else if (b.slmax > 0) loop_a_geo_2d<FRAC, true>(rec_sh, cls_sh, sl_sh, slg, lenr, uif, Df, Mf);
                else loop_a_geo_2d<FRAC, false>(rec_sh, cls_sh, sl_sh, slg, lenr, uif, Df, Mf);
            }
          }
        } else if (TILED) {
            const V4<R> me = tl_.pos[ms];
            const uint32_t pos_sh = tl::smem_u32(tl_.pos), rec_sh = tl::smem_u32(tl_.rec);
            const uint32_t sl_sh = tl::smem_u32(tl_.slots + (base - b.soff[p0 >> 5]) + lane * G);
            const uint16_t* slg = b.slots + base + lane * G;
            const bool staged = b.slmax > 0;
            const int lenr = b.wlen ? (int)b.wlen[w] : len;   // real longest row
            auto run = [&](auto U_, auto ST_) {
                constexpr bool U = decltype(U_)::value, ST = decltype(ST_)::value;
                if constexpr (sizeof(R) == 4 && DIM == 3)
                    loop_a_f2<FRAC, KIND, U, ST>(pos_sh, rec_sh, sl_sh, slg, lenr,
                                                 reinterpret_cast<const float4&>(me),
                                                 reinterpret_cast<const float4&>(ui), float(inv_h),
                                                 reinterpret_cast<float*>(D),
                                                 reinterpret_cast<float*>(M));
                else
                    loop_a<R, DIM, FRAC, KIND, U, ST>(pos_sh, rec_sh, sl_sh, slg, lenr, me, ui, inv_h,
                                                      D, M);
            };
            using T_ = std::true_type;
            using F_ = std::false_type;
            if (uni) {
                if (staged) run(T_{}, T_{}); else run(T_{}, F_{});
            } else {
                if (staged) run(F_{}, T_{}); else run(F_{}, F_{});
            }
        } else {
            const double xi = b.Xs[i], yi = b.Xs[N + i], zi = b.Xs[2 * N + i];
            const int32_t* sidx = b.sidx + base + lane;
            const double* __restrict__ Xp = b.Xs;
            const double* __restrict__ Yp = b.Xs + N;
            const double* __restrict__ Zp = b.Xs + 2 * N;
            // neighbours in groups of G: all index loads, then all gathers, then
            // the math, so each warp keeps 2G independent loads in flight
            for (int k = 0; k < len; k += G) {
                int32_t jj[G];
#pragma unroll
                for (int q = 0; q < G; ++q) jj[q] = __ldg(sidx + 32 * (k + q));
                double xj[G], yj[G], zj[G];
                V4<R> uj[G];
                R vj[G];
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    xj[q] = __ldg(Xp + jj[q]);
                    yj[q] = DIM == 3 ? __ldg(Yp + jj[q]) : 0.0;
                    zj[q] = __ldg(Zp + jj[q]);
                    uj[q] = tl::ldg4(us + 4 * (int64_t)jj[q]);
                    vj[q] = uni ? R(0) : R(__ldg(b.V0 + jj[q]));
                }
#pragma unroll
                for (int q = 0; q < G; ++q)
                    pair_a<R, DIM, FRAC, KIND>(R(xi - xj[q]), DIM == 3 ? R(yi - yj[q]) : R(0),
                                               R(zi - zj[q]), uj[q], vj[q], uni, ui, inv_h,
                                               D, M);
            }
        }
        pw = a_finish<R, DIM, MODEL, FRAC, KIND>(b, i, D, M, si, gated);
    }
    if (MODEL == 3) {
        // deterministic block partial of sum(dwp * V0)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
        if ((threadIdx.x & 31) == 0) s_pw[threadIdx.x >> 5] = pw;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_pw[k];
            b.pw_partial[tb] = t;
        }
    }
}

// ---------------------------------------------------------------------------
// boundary conditions (dynamics.py:159-217, fracture.py:46-83)
// ---------------------------------------------------------------------------
struct D3 {
    double x, y, z;
};

__device__ __forceinline__ void make_vars(tl::ExprVars& V, D3 X0, D3 u, double t, double dt,
                                          double dx) {
    V.v[0] = X0.x; V.v[1] = X0.y; V.v[2] = X0.z;
    V.v[3] = X0.x + u.x; V.v[4] = X0.y + u.y; V.v[5] = X0.z + u.z;
    V.v[6] = u.x; V.v[7] = u.y; V.v[8] = u.z;
    V.v[9] = t; V.v[10] = dt; V.v[11] = dx;
}

// the slice of tl_body the boundary-condition code needs, passed by value so
// out-of-line calls never copy the whole descriptor to local memory
struct BcCtx {
    const tl_bc* bcs;
    const tl_prog* progs;
    int64_t* counters;
    tl_clock* clock;
    double dp_body;
    int nbc, dim, restrict_prog;
};

__device__ __forceinline__ BcCtx bc_ctx(const tl_body& b) {
    return BcCtx{b.bcs, b.progs, b.counters, b.clock, b.dp_body, b.nbc, b.dim, b.restrict_prog};
}

__device__ __forceinline__ void note_err(const BcCtx& b, int err) {
    if (err) {
        atomicCAS((unsigned long long*)&b.counters[4], 0ull, (unsigned long long)err);
        flag_step_error(b.clock, 2);
    }
}

// a whole-body BC entry can apply during this step: the step evaluates BCs
// at times within [t, t + dt] (tl_body.bcw_lo/hi bound the entries' windows)
__device__ __forceinline__ bool whole_active(const tl_body& b) {
    if (!b.bc_whole) return false;
    const double t0 = b.clock ? b.clock->t : 0.0;
    const double dt = b.clock ? b.clock->dt : 0.0;
    return t0 <= b.bcw_hi && t0 + dt >= b.bcw_lo;
}

// some whole-body BC entry may act on particle i this step: its window meets
// [t, t + dt] and it has no skip guard valid for this step (t > gt) or the
// guard holds for i -- the same comparison the expression VM would make, on
// the same FP64 variables (make_vars), so the particles it skips are exactly
// those where every such entry evaluates to skip
template <typename R>
__device__ __forceinline__ bool whole_needed(const tl_body& b, int64_t i) {
    if (!whole_active(b)) return false;
    const double t0 = b.clock ? b.clock->t : 0.0;
    const double dt = b.clock ? b.clock->dt : 0.0;
    const int64_t N = b.n_all;
    for (int k = 0; k < b.nbc; ++k) {
        const tl_bc& c = b.bcs[k];
        if (c.bit >= 0 || t0 > c.tend || t0 + dt < c.tst) continue;
        if (c.gvar < 0 || !(t0 > c.gt)) return true;
        const int a = c.gvar % 3;
        double v;
        if (c.gvar < 3) {
            v = b.Xs[a * N + i];
        } else {
            const double u = double(static_cast<const R*>(b.us)[4 * i + a]);
            v = c.gvar < 6 ? b.Xs[a * N + i] + u : u;
        }
        const bool g = c.gop == 0 ? v < c.gc : (c.gop == 1 ? v > c.gc : (c.gop == 2 ? v <= c.gc : v >= c.gc));
        if (g) return true;
    }
    return false;
}

__device__ __forceinline__ bool bc_applies(const tl_bc& c, uint32_t mask, double t) {
    if (!(c.tst <= t && t <= c.tend)) return false;
    return c.bit < 0 || ((mask >> c.bit) & 1u);
}

// The BC evaluators are out of line and take / return plain values: the
// evaluator's stack lives in their own frames and the step kernels touch no
// local memory unless a particle actually carries a boundary condition.

// acc + force BCs active at t (file order), dynamics.py:159-190
__device__ __noinline__ D3 force_bcs(const BcCtx b, uint32_t mask, double m0i, D3 X0, D3 u,
                                     double t, double dt, D3 acc) {
    tl::ExprVars V;
    make_vars(V, X0, u, t, dt, b.dp_body);
    double a[3] = {acc.x, acc.y, acc.z};
    for (int k = 0; k < b.nbc; ++k) {
        const tl_bc c = b.bcs[k];
        if (c.kind != 1 || !bc_applies(c, mask, t)) continue;
        double scale = 1.0;
        if (c.ftype == 1) scale = 1.0 / m0i;
        else if (c.ftype == 2) scale = (b.dim == 3 ? b.dp_body * b.dp_body : b.dp_body) / m0i;
        for (int ax = 0; ax < 3; ++ax) {
            if (c.has_const[ax]) {
                a[ax] = tl::add_rn(a[ax], tl::mul_rn(c.cval[ax], scale));
            } else if (c.prog[ax] >= 0) {
                bool skip;
                int err = 0;
                const double val = tl::expr_eval(b.progs[c.prog[ax]], V, &skip, &err);
                note_err(b, err);
                a[ax] = tl::add_rn(a[ax], skip ? 0.0 : tl::mul_rn(val, scale));
            }
        }
    }
    return D3{a[0], a[1], a[2]};
}

// velocity components overwritten by velocity BCs active at t (file order),
// dynamics.py:193-217
__device__ __noinline__ D3 velocity_bcs(const BcCtx b, uint32_t mask, D3 X0, D3 u, double t,
                                        double dt, D3 vin) {
    tl::ExprVars V;
    make_vars(V, X0, u, t, dt, b.dp_body);
    double vel[3] = {vin.x, vin.y, vin.z};
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
    return D3{vel[0], vel[1], vel[2]};
}

// restrictphi floor (fracture.py:46-63); returns the floor or -1 for skip
__device__ __noinline__ double restrict_floor(const BcCtx b, D3 X0, D3 u, double t, double dt) {
    tl::ExprVars V;
    make_vars(V, X0, u, t, dt, b.dp_body);
    bool skip;
    int err = 0;
    const double val = tl::expr_eval(b.progs[b.restrict_prog], V, &skip, &err);
    note_err(b, err);
    if (skip) return -1.0;
    if (val < 0.0 || val > 1.0) {
        atomicExch((unsigned long long*)&b.counters[5], 1ull);
        flag_step_error(b.clock, 2);
    }
    return val;
}

// sdot += dtr*sddot; s += dts*sdot; clamp [0,1]; restrictphi floor
// (stepper.py:125-130, fracture.py:66-83)
// restrictphi applies to this particle: the expression is set and either
// its skip pattern is not static or the particle carries the restrict bit
// (the host found the expression non-skip there, simulation.py _setup_bcs)
__device__ __forceinline__ bool restrict_applies(const tl_body& b, uint32_t mask) {
    return b.restrict_prog >= 0 && (b.restrict_bit < 0 || ((mask >> b.restrict_bit) & 1u));
}

template <typename R, bool RESTRICT = true>
__device__ __forceinline__ void advance_phase(const tl_body& b, R& s, R& sd, R sdd, double dts,
                                              double dtr, D3 X0, D3 u, double t, double dt,
                                              uint32_t mask) {
    sd = tl::axpy_rn(sd, R(dtr), sdd);
    s = tl::axpy_rn(s, R(dts), sd);
    if (s < R(0)) { s = R(0); sd = R(0); }
    if (s > R(1)) { s = R(1); sd = R(0); }
    if (RESTRICT && restrict_applies(b, mask)) {
        const double fl = restrict_floor(bc_ctx(b), X0, u, t, dt);
        if (fl >= 0.0 && double(s) < fl) {
            s = R(fl);
            sd = R(0);
        }
    }
}

__device__ __forceinline__ double sq3_rn(double x, double y, double z) {
    // numpy einsum("nd,nd->n") order on (n,3): (x*x + z*z) + y*y
    return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(z, z)), __dmul_rn(y, y));
}

// Per-particle update after the force sum (stepper.py:86-130, dynamics.py:138-217,
// fracture.py:46-83): f0 and force BCs, the acceleration check, velocity BCs,
// the Verlet / symplectic kick and drift, the phase-field advance; writes
// v, u|s, sdot (and a when asked) and returns the dt maxima and the first
// non-finite particle.  BC = false is the common path: no boundary
// conditions and no restrictphi expression apply to this particle.
struct EpiOut {
    double v2, a2;
    long long bad;
};

template <typename R, int DIM, int MODE, bool FRAC, bool BC>
__device__ __forceinline__ EpiOut epi_body(const tl_body& b, int64_t i, uint32_t mask, double ax0,
                                           double ay0, double az0, R vi0, R vi1, R vi2) {
    EpiOut o{0.0, 0.0, LLONG_MAX};
    const int64_t N = b.n_all;
    double acc[3] = {ax0, ay0, az0};
    // a = (a_int + a_contact) + f0 + force BCs ; 2D a_y = 0  (stepper.py:86-95)
    if (b.ac) {
        acc[0] = tl::add_rn(acc[0], b.ac[i]);
        acc[1] = tl::add_rn(acc[1], b.ac[N + i]);
        acc[2] = tl::add_rn(acc[2], b.ac[2 * N + i]);
    }
    acc[0] = tl::add_rn(acc[0], b.f0[0]);
    acc[1] = tl::add_rn(acc[1], b.f0[1]);
    acc[2] = tl::add_rn(acc[2], b.f0[2]);
    const R* us = static_cast<const R*>(b.us);
    const auto ui = tl::ld4(us + 4 * i);
    const bool has_bc = BC && b.nbc && (mask || whole_needed<R>(b, i));
    const double t0 = b.clock ? b.clock->t : 0.0;
    const double dt = b.clock ? b.clock->dt : 0.0;
    const double tf = MODE == TL_B_INIT ? 0.0 : (MODE == TL_B_SYMPL ? t0 + 0.5 * dt : t0);
    const double dtf = MODE == TL_B_INIT ? 0.0 : dt;
    // reference positions only feed boundary-condition / restrictphi expressions
    const bool need_x = has_bc || (BC && FRAC && restrict_applies(b, mask));
    const D3 X0 = need_x ? D3{b.Xs[i], b.Xs[N + i], b.Xs[2 * N + i]} : D3{0.0, 0.0, 0.0};
    const D3 u0{double(ui.x), double(ui.y), double(ui.z)};
    if (has_bc) {
        const double m0i = b.uniform ? b.m0c : b.m0[i];
        const D3 r = force_bcs(bc_ctx(b), mask, m0i, X0, u0, tf, dtf, D3{acc[0], acc[1], acc[2]});
        acc[0] = r.x; acc[1] = r.y; acc[2] = r.z;
    }
    if (DIM == 2) acc[1] = 0.0;
    if (!(isfinite(acc[0]) && isfinite(acc[1]) && isfinite(acc[2]))) {
        o.bad = (long long)(b.perm ? b.perm[i] : i);
        if (b.clock) atomicMin((long long*)&b.counters[6], (long long)b.clock->step);
        flag_step_error(b.clock, 2);
    }
    // velocity: v_i is the copy pass A put in the record
    D3 vel{double(vi0), double(vi1), double(vi2)};
    R us_new[4] = {ui.x, ui.y, ui.z, ui.w};
    R* vout = static_cast<R*>(b.v);
    if (MODE == TL_B_INIT) {
        if (has_bc) vel = velocity_bcs(bc_ctx(b), mask, X0, u0, 0.0, 0.0, vel);
    } else {
        const double kick = MODE == TL_B_VERLET ? dt : 0.5 * dt;
        const double t_new = t0 + dt;
        // BC phase at the force time, kick, BCs at t_new, drift
        if (has_bc) vel = velocity_bcs(bc_ctx(b), mask, X0, u0, tf, dt, vel);
        vel = D3{double(tl::axpy_rn(R(vel.x), R(kick), R(acc[0]))),
                 double(tl::axpy_rn(R(vel.y), R(kick), R(acc[1]))),
                 double(tl::axpy_rn(R(vel.z), R(kick), R(acc[2])))};
        if (has_bc) vel = velocity_bcs(bc_ctx(b), mask, X0, u0, t_new, dt, vel);
        const R vR[3] = {R(vel.x), R(vel.y), R(vel.z)};
        us_new[0] = tl::axpy_rn(ui.x, R(kick), vR[0]);
        us_new[1] = DIM == 3 ? tl::axpy_rn(ui.y, R(kick), vR[1]) : R(0);
        us_new[2] = tl::axpy_rn(ui.z, R(kick), vR[2]);
        if (FRAC) {
            R* sdp = static_cast<R*>(b.sdot);
            R sd = sdp[i];
            R s = ui.w;
            const R sdd = static_cast<const R*>(b.sddot)[i];
            advance_phase<R, BC>(b, s, sd, sdd, kick, kick, X0,
                             D3{double(us_new[0]), double(us_new[1]), double(us_new[2])},
                             t_new, dt, mask);
            us_new[3] = s;
            sdp[i] = sd;
        }
        tl::st4(static_cast<R*>(b.us) + 4 * i, us_new[0], us_new[1], us_new[2], us_new[3]);
        if (b.peer_slot) {   // (u, s) into the neighbouring ranks' halo rows (NVLink)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int32_t slot = b.peer_slot[k * N + i];
                if (slot >= 0)
                    tl::st4(static_cast<R*>(b.peer_us[k]) + 4 * (int64_t)slot, us_new[0], us_new[1],
                            us_new[2], us_new[3]);
            }
        }
    }
    vout[i] = R(vel.x);
    vout[N + i] = R(vel.y);
    vout[2 * N + i] = R(vel.z);
    if (b.store_a || mirror_out(b)) {
        R* ap = static_cast<R*>(b.a);
#pragma unroll
        for (int a = 0; a < 3; ++a) ap[a * N + i] = R(acc[a]);
    }
    if (MODE != TL_B_INIT && b.clock &&
        !(isfinite(vel.x) && isfinite(vel.y) && isfinite(vel.z) && isfinite(double(us_new[0])) &&
          isfinite(double(us_new[1])) && isfinite(double(us_new[2])))) {
        atomicMin((long long*)&b.counters[7], (long long)b.clock->step + 1);
        b.clock->nf_now = 1;
    }
    const double vx = double(R(vel.x)), vy = double(R(vel.y)), vz = double(R(vel.z));
    const double ax = double(R(acc[0])), ay = double(R(acc[1])), az = double(R(acc[2]));
    o.v2 = sq3_rn(vx, vy, vz);
    o.a2 = sq3_rn(ax, ay, az);
    if (!(o.a2 == o.a2)) o.a2 = 0.0;  // NaN is reported through counters[3]
    if (!(o.v2 == o.v2)) o.v2 = 0.0;  // and through counters[7]
    return o;
}

template <typename R, int DIM, int MODE, bool FRAC>
__device__ __noinline__ EpiOut epi_slow(const tl_body* b, int64_t i, uint32_t mask, double ax,
                                        double ay, double az, R vi0, R vi1, R vi2) {
    return epi_body<R, DIM, MODE, FRAC, true>(*b, i, mask, ax, ay, az, vi0, vi1, vi2);
}

// ---------------------------------------------------------------------------
// pass B
// ---------------------------------------------------------------------------
// SPLIT > 1 (tiled FP32 3D, high-k stencils): SPLIT threads per member, part
// p summing the p-th share of the warp's slot groups; the shares are added in
// part order through shared memory and part 0 runs the epilogue.  A radial
// stencil's tile holds ~13 halo records per member, so shared memory allows
// one CTA per SM: the split gives it SPLIT times the warps to hide the
// shared-memory load latency of the pair loop.
// Pass B after the neighbour sums s1 = sum w r0, s2 = sum w PL_j r0, s3 =
// sum pi w r0 (without the kernel constant), shared by the tiled, L2-gather
// and brick kernels: the internal acceleration, then the particle's update
// (epi_body; the rare particles with BCs / restrictphi out of line).
template <typename R, int DIM, int MODE, bool FRAC, int KIND>
__device__ __forceinline__ EpiOut b_finish(const tl_body& b, int64_t i, R* s1, R* s2, R* s3,
                                           const R* PLi, R vi0, R vi1, R vi2) {
    const int64_t N = b.n_all;
    const bool uni = b.uniform != 0;
    const bool visc = b.visc != 0;
    const R inv_rho = R(1.0 / b.rho0);
    {   // kernel constant (and m0 when uniform), once per particle
        const R ck = kshape_const<R, KIND>(b) * (uni ? R(b.m0c) : R(1));
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            s1[q] *= ck;
            s2[q] *= ck;
            s3[q] *= ck * inv_rho;
        }
    }
    // a_int = (PL_i s1 + s2)/rho0^2 - AL_i s3
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
    // the rest of the particle's update: boundary conditions / restrictphi
    // expressions only on the (rare) particles that carry them, out of
    // line, so the common path holds no call frame
    const uint32_t mask = b.bcmask ? b.bcmask[i] : 0u;
    const bool slow = (b.nbc && (mask || whole_needed<R>(b, i))) || (FRAC && restrict_applies(b, mask));
    const EpiOut o = slow ? epi_slow<R, DIM, MODE, FRAC>(&b, i, mask, acc[0], acc[1], acc[2],
                                                         vi0, vi1, vi2)
                          : epi_body<R, DIM, MODE, FRAC, false>(b, i, mask, acc[0], acc[1],
                                                                acc[2], vi0, vi1, vi2);
    return o;
}

#ifndef TL_B_THREADS
#define TL_B_THREADS kThreads
#endif
template <int SPLIT>
constexpr int b_threads() { return SPLIT > 1 ? 1024 : TL_B_THREADS; }

template <typename R, int SPLIT>
constexpr int b_minb() { return SPLIT > 1 ? 1 : TL_MINB_B(R); }

template <typename R, int NREC>
__host__ __device__ constexpr size_t split_off(int S, int slmax) {
    return (tile_bytes<R, NREC>(S, slmax) + 15) & ~(size_t)15;
}

template <typename R, int DIM, int MODE, bool FRAC, int KIND, int G, bool TILED, int SPLIT = 1>
__global__ void __launch_bounds__(b_threads<SPLIT>(), b_minb<R, SPLIT>())
    k_pass_b(const __grid_constant__ tl_body b, const __grid_constant__ ClsTab<R> ct) {
    extern __shared__ __align__(16) unsigned char smem[];
    tl::pdl_enter();
    // a CTA of blockDim.x threads owns blockDim.x consecutive particles (TILED:
    // one shared tile of b.tile == blockDim.x particles); one particle per
    // thread -- larger tiles looped over by 256 threads measured slower
    // (shared memory per CTA cuts residency)
    const int T = SPLIT > 1 ? b.tile : (int)blockDim.x;
    const int64_t tb = tile_of(b, TILED);
    // L2 gather: lpp consecutive lanes per particle (tl_body.lpp), each summing
    // every lpp-th group of G slots of the row; the partial sums meet in a
    // butterfly, so every lane of a particle holds the same total
    const int lpp = TILED ? 1 : max(b.lpp, 1);
    const int sub = TILED ? 0 : (int)threadIdx.x & (lpp - 1);
    const int64_t p0 = tb * (int64_t)(T / lpp);
    if (halted(b) || stress_failed(b)) return;
    double v2 = 0.0, a2 = 0.0;
    long long bad_acc = LLONG_MAX;
    const R* rbp = static_cast<const R*>(b.rb);
    const bool uni = b.uniform != 0;
    Tile<R, 3> tl_;
    __shared__ uint64_t bar;
    if (TILED) {
        if (threadIdx.x == 32) prefetch_own_b<R, FRAC>(b, p0);
        tl_ = tile_layout<R, 3>(smem, b.tile + b.hmax, b.slmax, SPLIT == 1 ? b.ncls : 0);
        stage_tile<R, 3>(b, tl_, tb, b.tpos_b, rbp, &bar);
    }
    // 2D class-mode L2 gather: the class table's (W, kappa) entries in shared
    // memory (the per-lane class lookups of a constant-bank table measured
    // bimodal from launch to launch, 7.5-12.5 ms on C5)
    __shared__ V4<R> s_cls[(!TILED && DIM == 2) ? TL_TILE_MAX_CLASSES : 1];
    if constexpr (!TILED && DIM == 2) {
        if (b.ncls > 0 && b.bcls_host) {
            for (int c = threadIdx.x; c < b.ncls; c += blockDim.x) s_cls[c] = ct.W[c];
            __syncthreads();
        }
    }
    const int ms = SPLIT > 1 ? (int)threadIdx.x % T : (int)threadIdx.x / lpp;   // member slot
    const int part = SPLIT > 1 ? (int)threadIdx.x / T : 0;
    const bool live = p0 + ms < b.n;
    // SPLIT: every thread takes part in the share reduction; the dead ones of a
    // partial last tile read the last particle's row and sum nothing
    if (live || SPLIT > 1) {
        const int64_t i = live ? p0 + ms : b.n - 1;
        const int64_t N = b.n_all;
        const int lane = (int)(i & 31);
        const int64_t w = i >> 5;
        const int64_t base = b.soff[w];
        const int len = (int)((b.soff[w + 1] - base) >> 5);
        // own record: v_i now, P L_i after the neighbour loop (fewer live registers)
        const auto r2i = TILED ? tl_.rec[3 * ms + 2] : tl::ld4(rbp + 12 * i + 8);
        const R vi0 = r2i.x, vi1 = r2i.y, vi2 = r2i.z;
        const R inv_h = R(b.inv_h);
        const bool visc = b.visc != 0;
        const R eps_h2 = R(0.001 * b.h * b.h);
        const R B1 = R(b.beta1 * b.c0 * b.h), B2 = R(b.beta2 * b.h * b.h);
        const R inv_rho = R(1.0 / b.rho0);
        R s1[3] = {R(0), R(0), R(0)}, s2[3] = {R(0), R(0), R(0)}, s3[3] = {R(0), R(0), R(0)};
        if (TILED && SPLIT == 1 && tl_.cls != nullptr) {
          // bond classes: geometry from the class table, no positions
          const uint32_t rec_sh = tl::smem_u32(tl_.rec), cls_sh = tl::smem_u32(tl_.cls);
          const uint32_t sl_sh = tl::smem_u32(tl_.slots + (base - b.soff[p0 >> 5]) + lane * G);
          const uint16_t* slg = b.slots + base + lane * G;
          const int lenr = b.wlen ? (int)b.wlen[w] : len;
          if constexpr (sizeof(R) == 8) {
            double* d1 = reinterpret_cast<double*>(s1);
            double* d2 = reinterpret_cast<double*>(s2);
            double* d3 = reinterpret_cast<double*>(s3);
            const double B2d = double(B2), B1d = double(B1);
#define TL_LOOP_G64(ST, V, CC) loop_b_geo64<DIM, ST, V, CC>(rec_sh, cls_sh, sl_sh, slg, lenr, double(vi0), double(vi1), double(vi2), B2d, B1d, d1, d2, d3, reinterpret_cast<const ClsTab<double>*>(&ct))
            if (b.bcls_host && b.slmax > 0) {
                if (visc) TL_LOOP_G64(true, true, true); else TL_LOOP_G64(true, false, true);
            } else if (b.slmax > 0) {
                if (visc) TL_LOOP_G64(true, true, false); else TL_LOOP_G64(true, false, false);
            } else {
                if (visc) TL_LOOP_G64(false, true, false); else TL_LOOP_G64(false, false, false);
            }
#undef TL_LOOP_G64
          } else if constexpr (SPLIT == 1) {
            float* f1 = reinterpret_cast<float*>(s1);
            float* f2 = reinterpret_cast<float*>(s2);
            float* f3 = reinterpret_cast<float*>(s3);
            const float v0 = float(vi0), v1 = float(vi1), v2f = float(vi2);
            const float fB2 = float(B2), fB1 = float(B1);
#define TL_LOOP_G(ST, V, CC) loop_b_geo<DIM, ST, V, CC>(rec_sh, cls_sh, sl_sh, slg, lenr, v0, v1, v2f, fB2, fB1, f1, f2, f3, &ct)
            if (b.bcls_host && b.slmax > 0) {   // the common case: constant-bank classes
                if (visc) TL_LOOP_G(true, true, true); else TL_LOOP_G(true, false, true);
            } else if (b.slmax > 0) {
                if (visc) TL_LOOP_G(true, true, false); else TL_LOOP_G(true, false, false);
            } else {
                if (visc) TL_LOOP_G(false, true, false); else TL_LOOP_G(false, false, false);
            }
#undef TL_LOOP_G
          }
        } else if (TILED) {
            const V4<R> me = tl_.pos[ms];
            const uint32_t pos_sh = tl::smem_u32(tl_.pos), rec_sh = tl::smem_u32(tl_.rec);
            uint32_t sl_sh = tl::smem_u32(tl_.slots + (base - b.soff[p0 >> 5]) + lane * G);
            const uint16_t* slg = b.slots + base + lane * G;
            const bool staged = b.slmax > 0;
            int lenr = b.wlen ? (int)b.wlen[w] : len;   // real longest row
            if (SPLIT > 1) {   // this part's share of the warp's slot groups
                const int ng = (lenr + 3) >> 2;
                const int k0 = 4 * (ng * part / SPLIT), k1 = min(lenr, 4 * (ng * (part + 1) / SPLIT));
                sl_sh += 64u * (uint32_t)k0;
                slg += 32 * k0;
                lenr = live ? max(k1 - k0, 0) : 0;
            }
#define TL_LOOP_B(U, ST, V)                                                                        \
loop_b<R, DIM, KIND, U, ST, V>(pos_sh, rec_sh, sl_sh, slg, lenr, me, vi0, vi1, vi2, inv_h,    \
                               eps_h2, B2, B1, s1, s2, s3)
#define TL_LOOP_B2(U, ST)                                                                          \
if (visc) TL_LOOP_B(U, ST, true); else TL_LOOP_B(U, ST, false)
            if (uni) {
                if (staged) { TL_LOOP_B2(true, true); } else { TL_LOOP_B2(true, false); }
            } else {
                if (staged) { TL_LOOP_B2(false, true); } else { TL_LOOP_B2(false, false); }
            }
#undef TL_LOOP_B2
#undef TL_LOOP_B
        } else if (DIM == 2 && G == 4 && b.ncls > 0 && b.bcls_host && b.slots) {
            // L2 gather on a 2D lattice body with bond classes: the pair's class
            // is in the tiled layout's slot entry (same sliced shape, 2 bytes),
            // its (W, kappa) in the constant bank -- no position gathers and no
            // per-pair r or kernel shape.  The pair terms are loop_b_geo's
            // (loop_b_geo64's in FP64).
            const int32_t* sidx = b.sidx + base + lane;
            const uint16_t* slg = b.slots + base + lane * G;
            const R v0 = vi0, v2 = vi2;
            R a1x = R(0), a1z = R(0), a2x = R(0), a2z = R(0), a3x = R(0), a3z = R(0);
            for (int k = sub * G; k < len; k += G * lpp) {
                int32_t jj[G];
#pragma unroll
                for (int q = 0; q < G; ++q) jj[q] = __ldg(sidx + 32 * (k + q));
                const uint2 sg = __ldg(reinterpret_cast<const uint2*>(slg + 32 * k));
                const uint32_t e[G] = {sg.x & 0xffffu, sg.x >> 16, sg.y & 0xffffu, sg.y >> 16};
                V4<R> q0[G], q1[G], q2[G];
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    const R* rj = rbp + 12 * (int64_t)jj[q];
                    q0[q] = tl::ldg4(rj);
                    q1[q] = tl::ldg4(rj + 4);
                    q2[q] = tl::ldg4(rj + 8);
                }
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    const V4<R> W = s_cls[e[q] >> 10];
                    a1x += W.x; a1z += W.z;
                    a2x = fma(q1[q].x, W.z, fma(q0[q].x, W.x, a2x));
                    a2z = fma(q2[q].w, W.z, fma(q1[q].z, W.x, a2z));
                    if (visc) {
                        const R dvw = (v0 - q2[q].x) * W.x + (v2 - q2[q].z) * W.z;
                        const R g = dvw * W.w;
                        const R pw = (B2 * g - B1) * g;
                        a3x = fma(pw, W.x, a3x); a3z = fma(pw, W.z, a3z);
                    }
                }
            }
            s1[0] = a1x; s1[2] = a1z;
            s2[0] = a2x; s2[2] = a2z;
            s3[0] = a3x; s3[2] = a3z;
        } else {
            const double xi = b.Xs[i], yi = b.Xs[N + i], zi = b.Xs[2 * N + i];
            const int32_t* sidx = b.sidx + base + lane;
            const double* __restrict__ Xp = b.Xs;
            const double* __restrict__ Yp = b.Xs + N;
            const double* __restrict__ Zp = b.Xs + 2 * N;
            for (int k = sub * G; k < len; k += G * lpp) {
                int32_t jj[G];
#pragma unroll
                for (int q = 0; q < G; ++q) jj[q] = __ldg(sidx + 32 * (k + q));
                double xj[G], yj[G], zj[G];
                V4<R> q0[G], q1[G], q2[G];
                R mj[G];
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    xj[q] = __ldg(Xp + jj[q]);
                    yj[q] = DIM == 3 ? __ldg(Yp + jj[q]) : 0.0;
                    zj[q] = __ldg(Zp + jj[q]);
                    const R* rj = rbp + 12 * (int64_t)jj[q];
                    q0[q] = tl::ldg4(rj);
                    q1[q] = tl::ldg4(rj + 4);
                    q2[q] = tl::ldg4(rj + 8);
                    mj[q] = uni ? R(0) : R(__ldg(b.m0 + jj[q]));
                }
#pragma unroll
                for (int q = 0; q < G; ++q)
                    pair_b<R, DIM, KIND>(R(xi - xj[q]), DIM == 3 ? R(yi - yj[q]) : R(0),
                                         R(zi - zj[q]), q0[q], q1[q], q2[q], mj[q], uni, vi0, vi1,
                                         vi2, visc, inv_h, eps_h2, B2, B1, s1, s2, s3);
            }
        }
        if (lpp > 1) {   // a particle's lanes are live together (lpp divides 32)
            const unsigned am = __activemask();
            for (int o = 1; o < lpp; o <<= 1) {
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    s1[q] += __shfl_xor_sync(am, s1[q], o);
                    s2[q] += __shfl_xor_sync(am, s2[q], o);
                    s3[q] += __shfl_xor_sync(am, s3[q], o);
                }
            }
        }
        if constexpr (SPLIT > 1) {   // add the shares in part order
            R* red = reinterpret_cast<R*>(smem + split_off<R, 3>(b.tile + b.hmax, b.slmax));
            if (part > 0) {
                R* o = red + (size_t)(part - 1) * 9 * T + ms;
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    o[q * T] = s1[q];
                    o[(3 + q) * T] = s2[q];
                    o[(6 + q) * T] = s3[q];
                }
            }
            __syncthreads();
            if (part > 0) return;   // whole warps (T is a multiple of 32)
#pragma unroll 1
            for (int p = 1; p < SPLIT; ++p) {
                const R* o = red + (size_t)(p - 1) * 9 * T + ms;
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    s1[q] += o[q * T];
                    s2[q] += o[(3 + q) * T];
                    s3[q] += o[(6 + q) * T];
                }
            }
        }
        if (live && sub == 0) {   // the dead lanes of a split tile still join the warp reductions
            const auto r0i = TILED ? tl_.rec[3 * ms] : tl::ld4(rbp + 12 * i);
            const auto r1i = TILED ? tl_.rec[3 * ms + 1] : tl::ld4(rbp + 12 * i + 4);
            const R PLi[9] = {r0i.x, r0i.z, r1i.x, r0i.y, r0i.w, r1i.y, r1i.z, r1i.w, r2i.w};
            const EpiOut o = b_finish<R, DIM, MODE, FRAC, KIND>(b, i, s1, s2, s3, PLi, vi0, vi1, vi2);
            v2 = fmax(v2, o.v2);
            a2 = fmax(a2, o.a2);
            bad_acc = min(bad_acc, o.bad);
        }
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

// ---------------------------------------------------------------------------
// lattice-brick kernels (tl_body.brick): 3D lattice bodies with wide stencils
// ---------------------------------------------------------------------------
// A radial 3D stencil (k ~ 170) carries ~170 slot entries per particle in the
// tiled kernels -- more bytes than the particle's own state -- and a halo of
// ~13 records per member.  A body cut from one lattice needs neither: the
// CTA of a brick of lattice cells stages the records of the box of cells
// around it *by cell*, so a bond of class c (lattice offset q_c) is a fixed
// box offset from the member's cell, the same for every member.  Per
// particle only the bond mask (one bit per class, the reference CSR's
// membership: notches and body edges) is read; per pair a broadcast class
// load and the partner's records from shared memory.  Classes run in the
// reference's CSR order, so sums keep its summation order.
//
// Register blocking (tl_body.cpt = 2): a thread owns two cells adjacent in z.
// The classes of one (qx, qy) column of the stencil are consecutive in CSR
// order with qz descending, so the thread walks each column's partner cells
// once in ascending z and applies every record to both of its particles (the
// class of particle p against record k is qz = p - k): each particle still
// sums its bonds in CSR order, with about 40 % fewer shared-memory loads.
// Warps whose particles are not all complete (body edges, notches) take the
// per-bond path.
struct BrickGeo {
    int SX, SY, SZ, S;     // staged box (cells; SZ padded odd for cpt = 2)
    int ox, oy, oz;        // box origin (global cell)
    int tx, ty, tz;        // this thread's first member cell within the brick
};

__device__ __forceinline__ BrickGeo brick_geo(const tl_body& b, int64_t t, int cpt) {
    BrickGeo g;
    const int Rr = b.reach;
    g.SX = b.brick[0] + 2 * Rr;
    g.SY = b.brick[1] + 2 * Rr;
    g.SZ = b.boxz;
    g.S = g.SX * g.SY * g.SZ;
    const int bz = (int)(t % b.nbrick[2]);
    const int by = (int)((t / b.nbrick[2]) % b.nbrick[1]);
    const int bx = (int)(t / ((int64_t)b.nbrick[2] * b.nbrick[1]));
    g.ox = bx * b.brick[0] - Rr;
    g.oy = by * b.brick[1] - Rr;
    g.oz = bz * b.brick[2] - Rr;
    const int tid = (int)threadIdx.x;
    const int bzq = b.brick[2] / cpt;
    g.tz = (tid % bzq) * cpt;
    g.ty = (tid / bzq) % b.brick[1];
    g.tx = tid / (bzq * b.brick[1]);
    return g;
}

__device__ __forceinline__ int64_t cell_particle(const tl_body& b, int gx, int gy, int gz) {
    if (gx < 0 || gy < 0 || gz < 0 || gx >= b.cells[0] || gy >= b.cells[1] || gz >= b.cells[2])
        return -1;
    return b.cellmap[((int64_t)gx * b.cells[1] + gy) * b.cells[2] + gz];
}

// The class table rides in the kernel parameters (constant bank): the class
// loop is warp-uniform, so each class's W / U / box offset is one broadcast
// constant load with no shared-memory round trip ahead of the record loads.
template <typename R>
struct BrickTab {
    V4<R> W[TL_BRICK_MAX_CLASSES];   // (W, kappa)
    V4<R> U[TL_BRICK_MAX_CLASSES];   // (U, 0)
    int d[TL_BRICK_MAX_CLASSES];     // box-cell offset of the partner
    int4 col[TL_BRICK_MAX_COLUMNS];  // per (qx, qy) column: box offset, qz_lo, qz_hi, class of qz_hi
    int ncol;
};

// stage the NREC records of every occupied box cell (LDGSTS gathers; empty
// cells are never read)
template <typename R, int NREC>
__device__ __forceinline__ void stage_brick(const tl_body& b, const BrickGeo& g, const R* src,
                                            V4<R>* rec) {
    const int nt = (int)blockDim.x;
    constexpr int CH = (int)(sizeof(V4<R>) / 16) * NREC;   // 16-byte chunks per cell
    for (int sc = threadIdx.x; sc < g.S; sc += nt) {
        const int sz = sc % g.SZ, sy = (sc / g.SZ) % g.SY, sx = sc / (g.SZ * g.SY);
        const int64_t q = cell_particle(b, g.ox + sx, g.oy + sy, g.oz + sz);
        if (q >= 0) {
            const char* gp = reinterpret_cast<const char*>(src + q * 4 * NREC);
            char* sp = reinterpret_cast<char*>(rec + (int64_t)sc * NREC);
#pragma unroll
            for (int c = 0; c < CH; ++c) tl::cp_async16(sp + 16 * c, gp + 16 * c);
        }
    }
    tl::cp_async_wait_all();
    __syncthreads();
}

// every bond of particle i present (all mask bits of the body's classes)
__device__ __forceinline__ bool bonds_complete(const tl_body& b, int64_t i) {
    const int64_t N = b.n_all;
    const int nc = b.nbcls;
    bool full = true;
    for (int w = 0; w < b.nmask && full; ++w) {
        const int nb = min(32, nc - 32 * w);
        const uint32_t want = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
        full = b.bmask[w * N + i] == want;
    }
    return full;
}

// particle i's bonds in class order: a warp-uniform loop over the classes,
// predicated on the particle's mask bit (interior particles have every bit
// set; edges and notches clear some)
template <typename F>
__device__ __forceinline__ void each_bond(const tl_body& b, int64_t i, bool live, F&& pair) {
    const int64_t N = b.n_all;
    const int nc = b.nbcls;
    for (int w = 0; w < b.nmask; ++w) {
        const uint32_t m = live ? b.bmask[w * N + i] : 0u;
        const int cend = min(32, nc - 32 * w);
#pragma unroll 4
        for (int j = 0; j < cend; ++j)
            if ((m >> j) & 1u) pair(32 * w + j);
    }
}

// a thread's CPT particles against the stencil.  pair(p, c, o): particle p
// with class c and partner box cell o.  Complete warps walk the columns once
// (records shared by the CPT particles), the others bond by bond.
template <int CPT, typename R, typename F>
__device__ __forceinline__ void brick_bonds(const tl_body& b, const BrickTab<R>& tab,
                                            const int64_t* ip, const bool* live, int me0,
                                            F&& pair) {
    bool full = true;
#pragma unroll
    for (int p = 0; p < CPT; ++p) full = full && live[p] && bonds_complete(b, ip[p]);
    if (CPT > 1 && __all_sync(0xffffffffu, full)) {
        for (int cl = 0; cl < tab.ncol; ++cl) {
            const int4 col = tab.col[cl];   // (box offset, qz_lo, qz_hi, class of qz_hi)
            // partner of particle p for qz: me0 + p + col.x - qz, i.e. record k = p - qz
            for (int k = -col.z; k <= CPT - 1 - col.y; ++k) {
                const int o = me0 + col.x + k;
#pragma unroll
                for (int p = 0; p < CPT; ++p) {
                    const int qz = p - k;
                    if (qz >= col.y && qz <= col.z) pair(p, col.w + (col.z - qz), o);
                }
            }
        }
        return;
    }
#pragma unroll
    for (int p = 0; p < CPT; ++p)
        each_bond(b, ip[p], live[p], [&](int c) { pair(p, c, me0 + p + tab.d[c]); });
}

// FP32 packed pass-A accumulator (as loop_a_geo_f2)
struct AccA32 {
    float2 D01, D34, D67, D25, M01;
    float D8, M2, M3, M4, M5;
    float2 nui;
    float nuz, uis;
};

template <typename R, int MODEL, bool FRAC, int KIND, int CPT>
__global__ void __launch_bounds__(1024 / CPT, 1)
    k_brick_a(const __grid_constant__ tl_body b, const __grid_constant__ BrickTab<R> tab) {
    extern __shared__ __align__(16) unsigned char smem[];
    tl::pdl_enter();
    __shared__ double s_pw[32];
    if (halted(b)) return;
    const int64_t t = blockIdx.x;
    const BrickGeo g = brick_geo(b, t, CPT);
    V4<R>* rec = reinterpret_cast<V4<R>*>(smem);
    stage_brick<R, 1>(b, g, static_cast<const R*>(b.us), rec);
    const int me0 = ((g.tx + b.reach) * g.SY + g.ty + b.reach) * g.SZ + g.tz + b.reach;
    int64_t ip[CPT];
    bool live[CPT];
#pragma unroll
    for (int p = 0; p < CPT; ++p) {
        ip[p] = cell_particle(b, g.ox + b.reach + g.tx, g.oy + b.reach + g.ty,
                              g.oz + b.reach + g.tz + p);
        live[p] = ip[p] >= 0 && ip[p] < b.n;
    }
    double pw = 0.0;
    if constexpr (sizeof(R) == 4) {
        AccA32 A[CPT];
        const float4* rf = reinterpret_cast<const float4*>(rec);
#pragma unroll
        for (int p = 0; p < CPT; ++p) {
            const float4 ui = rf[me0 + p];
            A[p].D01 = A[p].D34 = A[p].D67 = A[p].D25 = A[p].M01 = make_float2(0.f, 0.f);
            A[p].D8 = A[p].M2 = A[p].M3 = A[p].M4 = A[p].M5 = 0.f;
            A[p].nui = make_float2(-ui.x, -ui.y);
            A[p].nuz = -ui.z;
            A[p].uis = ui.w;
        }
        brick_bonds<CPT>(b, tab, ip, live, me0, [&](int p, int c, int o) {
            AccA32& a = A[p];
            const float4 W = reinterpret_cast<const float4&>(tab.W[c]);
            const float4 uj = rf[o];
            const float2 wxy = make_float2(W.x, W.y);
            const float2 du01 = __fadd2_rn(make_float2(uj.x, uj.y), a.nui);
            const float du2 = uj.z + a.nuz;
            a.D01 = __ffma2_rn(make_float2(du01.x, du01.x), wxy, a.D01);
            a.D34 = __ffma2_rn(make_float2(du01.y, du01.y), wxy, a.D34);
            a.D67 = __ffma2_rn(make_float2(du2, du2), wxy, a.D67);
            a.D25 = __ffma2_rn(du01, make_float2(W.z, W.z), a.D25);
            a.D8 = fmaf(du2, W.z, a.D8);
            if (FRAC) {
                const float4 U = reinterpret_cast<const float4&>(tab.U[c]);
                const float ds = a.uis - uj.w;
                const float2 cw = __fmul2_rn(make_float2(ds, ds), wxy);
                const float cz = ds * W.z;
                a.M01 = __ffma2_rn(cw, make_float2(U.x, U.y), a.M01);
                a.M2 = fmaf(cz, U.z, a.M2);
                a.M3 = fmaf(cw.x, U.y, a.M3);
                a.M4 = fmaf(cw.x, U.z, a.M4);
                a.M5 = fmaf(cw.y, U.z, a.M5);
            }
        });
#pragma unroll
        for (int p = 0; p < CPT; ++p) {
            if (!live[p]) continue;
            const AccA32& a = A[p];
            R D[9] = {a.D01.x, a.D01.y, a.D25.x, a.D34.x, a.D34.y, a.D25.y, a.D67.x, a.D67.y, a.D8};
            R M[6] = {a.M01.x, a.M01.y, a.M2, a.M3, a.M4, a.M5};
            const R si = a.uis;
            pw += a_finish<R, 3, MODEL, FRAC, KIND>(b, ip[p], D, M, si, FRAC && si <= R(b.s_l));
        }
    } else {
        R D[CPT][9], M[CPT][6];
        V4<R> ui[CPT];
#pragma unroll
        for (int p = 0; p < CPT; ++p) {
            ui[p] = rec[me0 + p];
#pragma unroll
            for (int q = 0; q < 9; ++q) D[p][q] = R(0);
#pragma unroll
            for (int q = 0; q < 6; ++q) M[p][q] = R(0);
        }
        brick_bonds<CPT>(b, tab, ip, live, me0, [&](int p, int c, int o) {
            const V4<R> W = tab.W[c];
            const V4<R> uj = rec[o];
            R* Dp = D[p];
            R* Mp = M[p];
            const R du0 = uj.x - ui[p].x, du1 = uj.y - ui[p].y, du2 = uj.z - ui[p].z;
            Dp[0] = fma(du0, W.x, Dp[0]); Dp[1] = fma(du0, W.y, Dp[1]); Dp[2] = fma(du0, W.z, Dp[2]);
            Dp[3] = fma(du1, W.x, Dp[3]); Dp[4] = fma(du1, W.y, Dp[4]); Dp[5] = fma(du1, W.z, Dp[5]);
            Dp[6] = fma(du2, W.x, Dp[6]); Dp[7] = fma(du2, W.y, Dp[7]); Dp[8] = fma(du2, W.z, Dp[8]);
            if (FRAC) {
                const V4<R> U = tab.U[c];
                const R ds = ui[p].w - uj.w;
                const R cx = ds * W.x, cy = ds * W.y, cz = ds * W.z;
                Mp[0] = fma(cx, U.x, Mp[0]); Mp[1] = fma(cy, U.y, Mp[1]); Mp[2] = fma(cz, U.z, Mp[2]);
                Mp[3] = fma(cx, U.y, Mp[3]); Mp[4] = fma(cx, U.z, Mp[4]); Mp[5] = fma(cy, U.z, Mp[5]);
            }
        });
#pragma unroll
        for (int p = 0; p < CPT; ++p)
            if (live[p])
                pw += a_finish<R, 3, MODEL, FRAC, KIND>(b, ip[p], D[p], M[p], ui[p].w,
                                                        FRAC && ui[p].w <= R(b.s_l));
    }
    if (MODEL == 3) {   // deterministic CTA partial of sum(dwp * V0)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
        if ((threadIdx.x & 31) == 0) s_pw[threadIdx.x >> 5] = pw;
        __syncthreads();
        if (threadIdx.x == 0) {
            double acc = 0.0;
            for (int k = 0; k < (int)((blockDim.x + 31) >> 5); ++k) acc += s_pw[k];
            b.pw_partial[t] = acc;
        }
    }
}

// FP32 packed pass-B accumulator (as loop_b_geo)
struct AccB32 {
    float2 s1a, s2a, s3a, vi01;
    float s1b, s2b, s3b, vi2;
};

template <typename R, int MODE, bool FRAC, int KIND, int CPT>
__global__ void __launch_bounds__(1024 / CPT, 1)
    k_brick_b(const __grid_constant__ tl_body b, const __grid_constant__ BrickTab<R> tab) {
    extern __shared__ __align__(16) unsigned char smem[];
    tl::pdl_enter();
    if (halted(b) || stress_failed(b)) return;
    const int64_t t = blockIdx.x;
    const BrickGeo g = brick_geo(b, t, CPT);
    V4<R>* rec = reinterpret_cast<V4<R>*>(smem);
    stage_brick<R, 3>(b, g, static_cast<const R*>(b.rb), rec);
    const int me0 = ((g.tx + b.reach) * g.SY + g.ty + b.reach) * g.SZ + g.tz + b.reach;
    int64_t ip[CPT];
    bool live[CPT];
#pragma unroll
    for (int p = 0; p < CPT; ++p) {
        ip[p] = cell_particle(b, g.ox + b.reach + g.tx, g.oy + b.reach + g.ty,
                              g.oz + b.reach + g.tz + p);
        live[p] = ip[p] >= 0 && ip[p] < b.n;
    }
    const bool visc = b.visc != 0;
    const R B1 = R(b.beta1 * b.c0 * b.h), B2 = R(b.beta2 * b.h * b.h);
    R s1[CPT][3], s2[CPT][3], s3[CPT][3];
    if constexpr (sizeof(R) == 4) {
        const float4* rf = reinterpret_cast<const float4*>(rec);
        AccB32 A[CPT];
#pragma unroll
        for (int p = 0; p < CPT; ++p) {
            const float4 r2 = rf[3 * (me0 + p) + 2];
            A[p].s1a = A[p].s2a = A[p].s3a = make_float2(0.f, 0.f);
            A[p].s1b = A[p].s2b = A[p].s3b = 0.f;
            A[p].vi01 = make_float2(r2.x, r2.y);
            A[p].vi2 = r2.z;
        }
        const float2 neg1 = make_float2(-1.f, -1.f);
        const float fB1 = float(B1), fB2 = float(B2);
        auto run = [&](auto V_) {
            constexpr bool V = decltype(V_)::value;
            brick_bonds<CPT>(b, tab, ip, live, me0, [&](int p, int c, int oc) {
                AccB32& a = A[p];
                const float4 W = reinterpret_cast<const float4&>(tab.W[c]);
                const int o = 3 * oc;
                const float4 q0 = rf[o], q1 = rf[o + 1], q2 = rf[o + 2];
                const float2 wxy = make_float2(W.x, W.y);
                a.s1a = __fadd2_rn(a.s1a, wxy);
                a.s1b += W.z;
                a.s2a = __ffma2_rn(make_float2(q0.x, q0.y), make_float2(W.x, W.x), a.s2a);
                a.s2a = __ffma2_rn(make_float2(q0.z, q0.w), make_float2(W.y, W.y), a.s2a);
                a.s2a = __ffma2_rn(make_float2(q1.x, q1.y), make_float2(W.z, W.z), a.s2a);
                a.s2b = fmaf(q2.w, W.z, fmaf(q1.w, W.y, fmaf(q1.z, W.x, a.s2b)));
                if (V) {
                    const float2 dv = __ffma2_rn(make_float2(q2.x, q2.y), neg1, a.vi01);
                    const float2 pr = __fmul2_rn(dv, wxy);
                    const float dvw = fmaf(a.vi2 - q2.z, W.z, pr.x + pr.y);
                    const float gg = dvw * W.w;
                    const float pw = (fB2 * gg - fB1) * gg;
                    a.s3a = __ffma2_rn(make_float2(pw, pw), wxy, a.s3a);
                    a.s3b = fmaf(pw, W.z, a.s3b);
                }
            });
        };
        if (visc) run(std::true_type{}); else run(std::false_type{});
#pragma unroll
        for (int p = 0; p < CPT; ++p) {
            s1[p][0] = A[p].s1a.x; s1[p][1] = A[p].s1a.y; s1[p][2] = A[p].s1b;
            s2[p][0] = A[p].s2a.x; s2[p][1] = A[p].s2a.y; s2[p][2] = A[p].s2b;
            s3[p][0] = A[p].s3a.x; s3[p][1] = A[p].s3a.y; s3[p][2] = A[p].s3b;
        }
    } else {
        R vi[CPT][3];
#pragma unroll
        for (int p = 0; p < CPT; ++p) {
            const V4<R> r2 = rec[3 * (me0 + p) + 2];
            vi[p][0] = r2.x; vi[p][1] = r2.y; vi[p][2] = r2.z;
#pragma unroll
            for (int q = 0; q < 3; ++q) s1[p][q] = s2[p][q] = s3[p][q] = R(0);
        }
        brick_bonds<CPT>(b, tab, ip, live, me0, [&](int p, int c, int oc) {
            const V4<R> W = tab.W[c];
            const int o = 3 * oc;
            const V4<R> q0 = rec[o], q1 = rec[o + 1], q2 = rec[o + 2];
            R* a1 = s1[p];
            R* a2 = s2[p];
            R* a3 = s3[p];
            a1[0] += W.x; a1[1] += W.y; a1[2] += W.z;
            a2[0] = fma(q1.x, W.z, fma(q0.z, W.y, fma(q0.x, W.x, a2[0])));
            a2[1] = fma(q1.y, W.z, fma(q0.w, W.y, fma(q0.y, W.x, a2[1])));
            a2[2] = fma(q2.w, W.z, fma(q1.w, W.y, fma(q1.z, W.x, a2[2])));
            if (visc) {
                // explicit FMAs: one rounding sequence whatever the inlining context
                const R dvw = fma(vi[p][2] - q2.z, W.z, fma(vi[p][1] - q2.y, W.y, (vi[p][0] - q2.x) * W.x));
                const R gg = dvw * W.w;
                const R pw = fma(B2, gg, -B1) * gg;
                a3[0] = fma(pw, W.x, a3[0]); a3[1] = fma(pw, W.y, a3[1]); a3[2] = fma(pw, W.z, a3[2]);
            }
        });
    }
    double v2 = 0.0, a2 = 0.0;
    long long bad_acc = LLONG_MAX;
#pragma unroll
    for (int p = 0; p < CPT; ++p) {
        if (!live[p]) continue;
        const int me = me0 + p;
        const V4<R> r0i = rec[3 * me], r1i = rec[3 * me + 1], r2i = rec[3 * me + 2];
        const R PLi[9] = {r0i.x, r0i.z, r1i.x, r0i.y, r0i.w, r1i.y, r1i.z, r1i.w, r2i.w};
        const EpiOut o = b_finish<R, 3, MODE, FRAC, KIND>(b, ip[p], s1[p], s2[p], s3[p], PLi,
                                                          r2i.x, r2i.y, r2i.z);
        v2 = fmax(v2, o.v2);
        a2 = fmax(a2, o.a2);
        bad_acc = min(bad_acc, o.bad);
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

// ---------------------------------------------------------------------------
// opt-in hourglass control (tl_hourglass; include/tlsph.h)
// ---------------------------------------------------------------------------
template <typename R, int DIM, int KIND>
__global__ void __launch_bounds__(kThreads) k_hourglass(const tl_body b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (halted(b) || i >= b.n) return;
    const int64_t N = b.n_all;
    const R* Fh = static_cast<const R*>(b.Fh);
    const R* us = static_cast<const R*>(b.us);
    double Fi[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) Fi[q] = double(Fh[q * N + i]);
    const double Xi[3] = {b.Xs[i], b.Xs[N + i], b.Xs[2 * N + i]};
    const auto ui = tl::ld4(us + 4 * i);
    const double xi[3] = {Xi[0] + double(ui.x), Xi[1] + double(ui.y), Xi[2] + double(ui.z)};
    const int lane = (int)(i & 31);
    const int64_t w = i >> 5;
    const int64_t base = b.soff[w];
    const int len = (int)((b.soff[w + 1] - base) >> 5);
    const int32_t* sidx = b.sidx + base + lane;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < len; ++k) {
        const int64_t j = sidx[32 * k];
        if (j == i) continue;                 // row padding
        double Xij[3], xij[3], Fj[9];
#pragma unroll
        for (int a = 0; a < 3; ++a) Xij[a] = b.Xs[a * N + j] - Xi[a];
        const auto uj = tl::ld4(us + 4 * j);
        xij[0] = Xij[0] + double(uj.x) - double(ui.x);
        xij[1] = Xij[1] + double(uj.y) - double(ui.y);
        xij[2] = Xij[2] + double(uj.z) - double(ui.z);
        if (DIM == 2) { Xij[1] = 0.0; xij[1] = 0.0; }
#pragma unroll
        for (int q = 0; q < 9; ++q) Fj[q] = double(Fh[q * N + j]);
        const double R2 = Xij[0] * Xij[0] + Xij[1] * Xij[1] + Xij[2] * Xij[2];
        const double r = sqrt(xij[0] * xij[0] + xij[1] * xij[1] + xij[2] * xij[2]);
        if (!(r > 0.0) || !(R2 > 0.0)) continue;
        const double Rn = sqrt(R2);
        // kernel value W(|X_ij|) (kernel_geom.py:30-62)
        const double q = Rn * b.inv_h;
        double Wv;
        if (KIND == 2) {
            const double t = fmax(1.0 - 0.5 * q, 0.0);
            Wv = b.alpha * t * t * t * t * (2.0 * q + 1.0);
        } else {
            const double tm = 2.0 - q;
            Wv = b.alpha * (q < 1.0 ? 1.0 - 1.5 * q * q + 0.75 * q * q * q
                                    : (q < 2.0 ? 0.25 * tm * tm * tm : 0.0));
        }
        double di = 0.0, dj = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double pi_ = Fi[3 * a] * Xij[0] + Fi[3 * a + 1] * Xij[1] + Fi[3 * a + 2] * Xij[2];
            const double pj_ = Fj[3 * a] * Xij[0] + Fj[3 * a + 1] * Xij[1] + Fj[3 * a + 2] * Xij[2];
            di += (pi_ - xij[a]) * xij[a];
            dj += (pj_ - xij[a]) * xij[a];
        }
        const double Vj = b.uniform ? b.V0c : b.V0[j];
        // a_i += -(alpha E / (2 rho0)) V_j W / |X|^2 (d_ij + d_ji) x_ij / |x_ij|, with
        // d = (F X_ij - x_ij) . x_ij / |x_ij|
        const double c = -b.hg_coef * Vj * Wv / R2 * (di + dj) / (r * r);
#pragma unroll
        for (int a = 0; a < 3; ++a) acc[a] += c * xij[a];
    }
    double* ac = const_cast<double*>(b.ac);
    ac[i] += acc[0];
    ac[N + i] += DIM == 2 ? 0.0 : acc[1];
    ac[2 * N + i] += acc[2];
}

// symplectic predictor (stepper.py:168-175)
template <typename R, int DIM, bool FRAC>
__global__ void __launch_bounds__(kThreads) k_predict(const tl_body b) {
    tl::pdl_enter();
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
    D3 vel{double(tl::axpy_rn(vp[i], R(half), ap[i])), double(tl::axpy_rn(vp[N + i], R(half), ap[N + i])),
           double(tl::axpy_rn(vp[2 * N + i], R(half), ap[2 * N + i]))};
    const uint32_t mask = b.bcmask ? b.bcmask[i] : 0u;
    const D3 X0{xi, yi, zi};
    if (b.nbc && (mask || whole_needed<R>(b, i)))
        vel = velocity_bcs(bc_ctx(b), mask, X0, D3{double(ui.x), double(ui.y), double(ui.z)}, th, dt, vel);
    R vR[3] = {R(vel.x), R(vel.y), R(vel.z)};
    R un[4] = {tl::axpy_rn(ui.x, R(half), vR[0]), DIM == 3 ? tl::axpy_rn(ui.y, R(half), vR[1]) : R(0),
               tl::axpy_rn(ui.z, R(half), vR[2]), ui.w};
    if (FRAC) {
        R* sdp = static_cast<R*>(b.sdot);
        R sd = sdp[i], s = ui.w;
        advance_phase<R>(b, s, sd, static_cast<const R*>(b.sddot)[i], half, half, X0,
                         D3{double(un[0]), double(un[1]), double(un[2])}, th, dt, mask);
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
    tl::pdl_enter();
    // every word the clock reads, loaded up front: one memory round trip
    // instead of a chain of dependent ones (the kernel is on the critical
    // path of every step)
    const tl_clock cl = *c;
    unsigned long long rv[8], ra[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        rv[k] = k < info.n ? info.d[k].red[0] : 0ull;
        ra[k] = k < info.n ? info.d[k].red[1] : 0ull;
    }
    if (cl.halted) return;
    if (cl.err) {          // the previous step raised: nothing more runs
        c->halted = 5;
        return;
    }
    c->nf_now = 0;
    if (!(cl.t < cl.t_max - cl.eps)) {
        c->halted = 1;
        return;
    }
    double dt;
    if (cl.dt_override >= 0.0) {
        dt = cl.dt_override;
    } else {
        dt = INFINITY;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (k >= info.n) break;
            const double vmax = sqrt(__longlong_as_double((long long)rv[k]));
            const double amax = sqrt(__longlong_as_double((long long)ra[k]));
            const double dtv = info.d[k].h / (info.d[k].c0 + vmax);
            double cand = amax > 0.0 ? cl.cfl * fmin(dtv, sqrt(info.d[k].h / amax)) : cl.cfl * dtv;
            // a NaN maximum (non-finite state) must stop the clock, not vanish in fmin
            dt = (isnan(cand) || cand < dt) ? cand : dt;
        }
    }
    dt = fmin(fmin(dt, cl.next_out - cl.t), cl.t_max - cl.t);
    if (!(dt > 0.0) || isinf(dt)) {
        c->halted = 4;
        c->dt = dt;
        return;
    }
    c->dt = dt;
    // the maxima are read: clear them for this step's pass B (replaces a
    // memset node per body per step)
    for (int k = 0; k < info.n; ++k) {
        info.d[k].red[0] = 0ull;
        info.d[k].red[1] = 0ull;
    }
    const double tn = cl.t + dt;
    c->out_step = (tn >= cl.next_out - cl.eps) || (tn >= cl.t_max - cl.eps) ||
                  (cl.max_steps >= 0 && cl.step + 1 >= cl.max_steps);
}

__global__ void k_clock_commit(tl_clock* c) {
    tl::pdl_enter();
    const tl_clock cl = *c;            // one round trip (see k_clock_begin)
    if (cl.halted || cl.err) return;   // a step that raised is not committed
    const double t = cl.t + cl.dt;
    const int64_t step = cl.step + 1;
    c->t = t;
    c->step = step;
    // stepper.py:203-209: the state check of every 64th commit
    if (step % 64 == 0 && cl.nf_now) c->halted = 6;
    else if (t >= cl.next_out - cl.eps) c->halted = 2;
    else if (cl.max_steps >= 0 && step >= cl.max_steps) c->halted = 3;
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
// dynamic shared memory of the tiled kernels; opted in once per kernel
template <typename K>
int smem_opt_in(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return TL_OK;
    if (bytes > 227 * 1024) {
        tl_set_error("tile needs %zu bytes of shared memory", bytes);
        return TL_ERR_ARG;
    }
    TL_TRY_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return TL_OK;
}

template <typename R, typename K>
int launch_brick(K kern, cudaStream_t st, const tl_body& b, int nrec) {
    const int cpt = b.cpt > 0 ? b.cpt : 1;
    const int T = b.brick[0] * b.brick[1] * b.brick[2] / cpt;
    if (T <= 0 || T > 1024 / cpt || T % 32 || b.brick[2] % cpt || b.nbcls <= 0 ||
        b.nbcls > TL_BRICK_MAX_CLASSES || b.nmask <= 0 || b.nmask * 32 < b.nbcls ||
        !b.bdelta_host || !b.bbcls_host || b.boxz < b.brick[2] + 2 * b.reach ||
        (cpt > 1 && (b.ncol <= 0 || b.ncol > TL_BRICK_MAX_COLUMNS || !b.bcol_host))) {
        tl_set_error("tl_body: invalid brick descriptor");
        return TL_ERR_ARG;
    }
    BrickTab<R> tab;
    const V4<R>* hc = static_cast<const V4<R>*>(b.bbcls_host);
    for (int c = 0; c < TL_BRICK_MAX_CLASSES; ++c) {
        if (c < b.nbcls) {
            tab.W[c] = hc[2 * c];
            tab.U[c] = hc[2 * c + 1];
            tab.d[c] = b.bdelta_host[c];
        } else {
            tab.W[c] = tab.U[c] = V4<R>{};
            tab.d[c] = 0;
        }
    }
    tab.ncol = cpt > 1 ? b.ncol : 0;
    for (int c = 0; c < TL_BRICK_MAX_COLUMNS; ++c)
        tab.col[c] = (c < tab.ncol) ? make_int4(b.bcol_host[4 * c], b.bcol_host[4 * c + 1],
                                                b.bcol_host[4 * c + 2], b.bcol_host[4 * c + 3])
                                    : make_int4(0, 0, -1, 0);
    const int S = (b.brick[0] + 2 * b.reach) * (b.brick[1] + 2 * b.reach) * b.boxz;
    const size_t bytes = (size_t)S * nrec * sizeof(V4<R>);
    int rc = smem_opt_in(kern, bytes);
    if (rc) return rc;
    const int64_t nb = (int64_t)b.nbrick[0] * b.nbrick[1] * b.nbrick[2];
    TL_TRY_CUDA(tl_launch(kern, dim3((unsigned)nb), dim3(T), bytes, st, b, tab));
    return TL_OK;
}

template <typename R, int DIM, int MODEL, bool FRAC, int KIND>
int launch_a_one(cudaStream_t st, const tl_body& b) {
    constexpr int G = TL_GATHER_A;
    if constexpr (DIM == 3) {
        if (b.brick[0] > 0) {
            tl_body ba = b;       // pass A may run smaller bricks (same box offsets)
            if (b.a_split > 1 && b.brick[0] % b.a_split == 0) {
                ba.brick[0] = b.brick[0] / b.a_split;
                ba.nbrick[0] = (b.cells[0] + ba.brick[0] - 1) / ba.brick[0];
            }
            int rc = b.cpt == 2 ? launch_brick<R>(k_brick_a<R, MODEL, FRAC, KIND, 2>, st, ba, 1)
                                : launch_brick<R>(k_brick_a<R, MODEL, FRAC, KIND, 1>, st, ba, 1);
            return rc ? rc : tl_check_launch("k_brick_a");
        }
    }
    if (b.tile > kThreads || (b.tile > 0 && b.tile % 32)) {
        tl_set_error("tile %d: pass A needs a multiple of 32, at most %d", b.tile, kThreads);
        return TL_ERR_ARG;
    }
    ClsTabA<R> ct{};   // the class table for the constant bank (tl_body.bcls_host)
    if (b.tile > 0 && b.ncls > 0 && b.bcls_host) {
        if (b.ncls > TL_TILE_MAX_CLASSES) {
            tl_set_error("%d bond classes: at most %d", b.ncls, TL_TILE_MAX_CLASSES);
            return TL_ERR_ARG;
        }
        const R* hc = static_cast<const R*>(b.bcls_host);
        for (int c = 0; c < b.ncls; ++c) {
            ct.W[c] = V4<R>{hc[8 * c], hc[8 * c + 1], hc[8 * c + 2], hc[8 * c + 3]};
            ct.U[c] = V4<R>{hc[8 * c + 4], hc[8 * c + 5], hc[8 * c + 6], hc[8 * c + 7]};
        }
    }
    if (b.tile > 0) {
        auto kern = k_pass_a<R, DIM, MODEL, FRAC, KIND, G, true>;
        const size_t bytes = tile_bytes<R, 1>(b.tile + b.hmax, b.slmax, b.ncls);
        int rc = smem_opt_in(kern, bytes);
        if (rc) return rc;
        TL_TRY_CUDA(tl_launch(kern, dim3(b.tlist ? (unsigned)b.tcount : tl_blocks(b.n, b.tile)),
                              dim3(b.tile), bytes, st, b, ct));
    } else {
        TL_TRY_CUDA(tl_launch(k_pass_a<R, DIM, MODEL, FRAC, KIND, G, false>,
                              dim3(tl_blocks(b.n, kThreads)), dim3(kThreads), 0, st, b, ct));
    }
    return tl_check_launch("k_pass_a");
}

template <typename R, int DIM, int KIND>
int launch_a_k(cudaStream_t st, const tl_body& b) {
    if (b.model == 1)
        return b.fracture ? launch_a_one<R, DIM, 1, true, KIND>(st, b) : launch_a_one<R, DIM, 1, false, KIND>(st, b);
    if (b.model == 2)
        return b.fracture ? launch_a_one<R, DIM, 2, true, KIND>(st, b) : launch_a_one<R, DIM, 2, false, KIND>(st, b);
    return launch_a_one<R, DIM, 3, false, KIND>(st, b);
}

template <typename R, int DIM>
int launch_a(cudaStream_t st, const tl_body& b) {
    return b.kind == 1 ? launch_a_k<R, DIM, 1>(st, b) : launch_a_k<R, DIM, 2>(st, b);
}

template <typename R, int DIM, int MODE, bool FRAC, int KIND>
int launch_b_one(cudaStream_t st, const tl_body& b) {
    constexpr int G = TL_GATHER_B;
    if constexpr (DIM == 3) {
        if (b.brick[0] > 0) {
            int rc = b.cpt == 2 ? launch_brick<R>(k_brick_b<R, MODE, FRAC, KIND, 2>, st, b, 3)
                                : launch_brick<R>(k_brick_b<R, MODE, FRAC, KIND, 1>, st, b, 3);
            return rc ? rc : tl_check_launch("k_brick_b");
        }
    }
    // the class table's (W, kappa) entries for the constant bank (tl_body.bcls_host)
    ClsTab<R> ct{};   // also for the L2 gather (tile 0), whose 2D class mode reads it
    if (b.ncls > 0 && b.bcls_host) {
        if (b.ncls > TL_TILE_MAX_CLASSES) {
            tl_set_error("%d bond classes: at most %d", b.ncls, TL_TILE_MAX_CLASSES);
            return TL_ERR_ARG;
        }
        const R* hc = static_cast<const R*>(b.bcls_host);
        for (int c = 0; c < b.ncls; ++c)
            ct.W[c] = V4<R>{hc[8 * c], hc[8 * c + 1], hc[8 * c + 2], hc[8 * c + 3]};
    }
    if constexpr (sizeof(R) == 4 && DIM == 3) {
        if (b.tile > 0 && b.bsplit == 4) {
            constexpr int SP = 4;
            if (b.tile * SP > 1024) {
                tl_set_error("bsplit %d needs tile <= %d", SP, 1024 / SP);
                return TL_ERR_ARG;
            }
            if (b.ncls > 0) {
                tl_set_error("bsplit 4 with bond classes (slot entries carry a class)");
                return TL_ERR_ARG;
            }
            auto kern = k_pass_b<R, DIM, MODE, FRAC, KIND, G, true, SP>;
            const size_t bytes = split_off<R, 3>(b.tile + b.hmax, b.slmax) +
                                 (size_t)(SP - 1) * 9 * b.tile * sizeof(R);
            int rc = smem_opt_in(kern, bytes);
            if (rc) return rc;
            TL_TRY_CUDA(tl_launch(kern, dim3(b.tlist ? (unsigned)b.tcount : tl_blocks(b.n, b.tile)),
                                  dim3(b.tile * SP), bytes, st, b, ct));
            return tl_check_launch("k_pass_b");
        }
    }
    if (b.tile > 0 && b.bsplit > 1) {
        tl_set_error("bsplit: tiled FP32 3D pass B only (bsplit 4)");
        return TL_ERR_ARG;
    }
    if (b.tile > kThreads || (b.tile > 0 && b.tile % 32)) {
        tl_set_error("tile %d: pass B needs a multiple of 32, at most %d", b.tile, kThreads);
        return TL_ERR_ARG;
    }
    if (b.tile > 0) {
        auto kern = k_pass_b<R, DIM, MODE, FRAC, KIND, G, true>;
        const size_t bytes = tile_bytes<R, 3>(b.tile + b.hmax, b.slmax, b.ncls);
        int rc = smem_opt_in(kern, bytes);
        if (rc) return rc;
        TL_TRY_CUDA(tl_launch(kern, dim3(b.tlist ? (unsigned)b.tcount : tl_blocks(b.n, b.tile)),
                              dim3(b.tile), bytes, st, b, ct));
    } else {
        const int lpp = max(b.lpp, 1);
        if (lpp > 8 || (lpp & (lpp - 1))) {
            tl_set_error("lpp %d: 1, 2, 4 or 8 lanes per particle", lpp);
            return TL_ERR_ARG;
        }
        TL_TRY_CUDA(tl_launch(k_pass_b<R, DIM, MODE, FRAC, KIND, G, false>,
                              dim3(tl_blocks(b.n * lpp, kThreads)), dim3(kThreads), 0, st, b, ct));
    }
    return tl_check_launch("k_pass_b");
}

template <typename R, int DIM, int MODE, int KIND>
int launch_b_mode(cudaStream_t st, const tl_body& b) {
    return b.fracture ? launch_b_one<R, DIM, MODE, true, KIND>(st, b)
                      : launch_b_one<R, DIM, MODE, false, KIND>(st, b);
}

template <typename R, int DIM, int KIND>
int launch_b_k(cudaStream_t st, const tl_body& b, int mode) {
    if (mode == TL_B_INIT) return launch_b_mode<R, DIM, TL_B_INIT, KIND>(st, b);
    if (mode == TL_B_VERLET) return launch_b_mode<R, DIM, TL_B_VERLET, KIND>(st, b);
    return launch_b_mode<R, DIM, TL_B_SYMPL, KIND>(st, b);
}

template <typename R, int DIM>
int launch_b(cudaStream_t st, const tl_body& b, int mode) {
    return b.kind == 1 ? launch_b_k<R, DIM, 1>(st, b, mode) : launch_b_k<R, DIM, 2>(st, b, mode);
}

template <typename R, int DIM>
int launch_p(cudaStream_t st, const tl_body& b) {
    const unsigned g = tl_blocks(b.n, kThreads);
    if (b.fracture) TL_TRY_CUDA(tl_launch(k_predict<R, DIM, true>, dim3(g), dim3(kThreads), 0, st, b));
    else TL_TRY_CUDA(tl_launch(k_predict<R, DIM, false>, dim3(g), dim3(kThreads), 0, st, b));
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

// FP64 SVK split of the fused pass A on caller-given strains (test hook):
// the closed form where it applies, the cyclic Jacobi elsewhere
__global__ void k_svk_split_check(int64_t n, const double* H, double lam, double mu, const double* s,
                                  double* S, double* psi, double* psip, int32_t* closed) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double h[9], Sv[9], ps, pp;
#pragma unroll
    for (int k = 0; k < 9; ++k) h[k] = H[9 * i + k];
    svk_update<double>(h, lam, mu, s[i], true, 1e-30, Sv, ps, pp);
#pragma unroll
    for (int k = 0; k < 9; ++k) S[9 * i + k] = Sv[k];
    psi[i] = ps;
    psip[i] = pp;
    double E[9], Ep[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            E[3 * r + c] = 0.5 * (h[3 * r + c] + h[3 * c + r] +
                                  (h[r] * h[c] + h[3 + r] * h[3 + c] + h[6 + r] * h[6 + c]));
    closed[i] = positive_part64(E, Ep) ? 1 : 0;
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
    TL_TRY_CUDA(tl_launch(k_clock_begin, dim3(1), dim3(1), 0, (cudaStream_t)st, clock, d));
    return tl_check_launch("k_clock_begin");
}

extern "C" int tl_clock_commit(tl_stream_t st, tl_clock* clock) {
    TL_TRY_CUDA(tl_launch(k_clock_commit, dim3(1), dim3(1), 0, (cudaStream_t)st, clock));
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

extern "C" int tl_svk_split_check(tl_stream_t st, int64_t n, const double* H, double lam, double mu,
                                  const double* s, double* S, double* psi, double* psip,
                                  int32_t* closed) {
    if (n <= 0) return TL_OK;
    k_svk_split_check<<<tl_blocks(n, kThreads), kThreads, 0, (cudaStream_t)st>>>(n, H, lam, mu, s, S,
                                                                                psi, psip, closed);
    return tl_check_launch("k_svk_split_check");
}

extern "C" int tl_hourglass(tl_stream_t st_, const tl_body* b) {
    int rc = check_body(b);
    if (rc) return rc;
    if (!b->Fh || !b->ac) {
        tl_set_error("tl_hourglass: needs the F planes (Fh) and the acceleration planes (ac)");
        return TL_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)st_;
    const unsigned g = tl_blocks(b->n, kThreads);
    if (b->precision == 4) {
        if (b->dim == 3) {
            if (b->kind == 2) k_hourglass<float, 3, 2><<<g, kThreads, 0, st>>>(*b);
            else k_hourglass<float, 3, 1><<<g, kThreads, 0, st>>>(*b);
        } else {
            if (b->kind == 2) k_hourglass<float, 2, 2><<<g, kThreads, 0, st>>>(*b);
            else k_hourglass<float, 2, 1><<<g, kThreads, 0, st>>>(*b);
        }
    } else {
        if (b->dim == 3) {
            if (b->kind == 2) k_hourglass<double, 3, 2><<<g, kThreads, 0, st>>>(*b);
            else k_hourglass<double, 3, 1><<<g, kThreads, 0, st>>>(*b);
        } else {
            if (b->kind == 2) k_hourglass<double, 2, 2><<<g, kThreads, 0, st>>>(*b);
            else k_hourglass<double, 2, 1><<<g, kThreads, 0, st>>>(*b);
        }
    }
    return tl_check_launch("k_hourglass");
}
