// output.cu -- device-side output reductions.
//
// The reference computes its output rows on the host from the full particle
// state: compute_energies (output.py:25-49) -- strain V0.psi_e, kinetic
// 1/2 m0 |v|^2, fracture surface energy with the corrected SPH gradient of s
// (backends/fast.py:156-169) -- and measure_row (output.py:63-71) -- mean
// displacement and total force m0*a over a measure-plane set.  At 16M-128M
// particles that is a multi-GB device->host copy per output; here each
// quantity is reduced on the device into per-block FP64 partials (fixed
// block order, deterministic), which the host adds with math.fsum.
#include "tl_common.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double sq3_rn(double x, double y, double z) {
    // numpy einsum("nd,nd->n") order on (n,3): (x*x + z*z) + y*y
    return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(z, z)), __dmul_rn(y, y));
}

// deterministic block sum of NV values per thread -> out[blockIdx.x * NV + k]
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* out) {
    __shared__ double sh[NV][kThreads / 32];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[threadIdx.x][w];
        out[(int64_t)blockIdx.x * NV + threadIdx.x] = t;
    }
}

// (strain, kinetic, fracture) energy partials over the owned particles
template <typename R, int DIM, int KIND>
__global__ void __launch_bounds__(kThreads) k_energies(const tl_body b, double* part) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double acc[3] = {0.0, 0.0, 0.0};
    if (i < b.n) {
        const int64_t N = b.n_all;
        const double V0i = b.uniform ? b.V0c : b.V0[i];
        const double m0i = b.uniform ? b.m0c : b.m0[i];
        acc[0] = V0i * b.psi_out[i];
        const R* v = static_cast<const R*>(b.v);
        acc[1] = 0.5 * m0i * sq3_rn(double(v[i]), double(v[N + i]), double(v[2 * N + i]));
        if (b.fracture) {
            // grad s_i = L_i sum_j V0_j (s_j - s_i) fac_ij r0_ij   (CSR order)
            const R* us = static_cast<const R*>(b.us);
            const double si = double(us[4 * i + 3]);
            const double xi = b.Xs[i], yi = b.Xs[N + i], zi = b.Xs[2 * N + i];
            const double inv_h = b.inv_h, a_ih = b.alpha * b.inv_h;
            double g[3] = {0.0, 0.0, 0.0};
            const int lane = (int)(i & 31);
            const int64_t w = i >> 5;
            const int64_t base = b.soff[w];
            const int len = (int)((b.soff[w + 1] - base) >> 5);
            for (int k = 0; k < len; ++k) {
                const int64_t j = b.sidx[base + 32 * k + lane];
                if (j == i) continue;   // padding (self)
                const double dx = xi - b.Xs[j], dy = DIM == 3 ? yi - b.Xs[N + j] : 0.0,
                             dz = zi - b.Xs[2 * N + j];
                const double r2 = dx * dx + dy * dy + dz * dz;
                const double fac = tl::kernel_fac<double, KIND>(r2, tl::rsqrt_pos(r2), inv_h, a_ih);
                const double V0j = b.uniform ? b.V0c : b.V0[j];
                const double c = V0j * (double(us[4 * j + 3]) - si) * fac;
                g[0] += c * dx;
                g[1] += c * dy;
                g[2] += c * dz;
            }
            const R* L = static_cast<const R*>(b.L);
            double gr[3];
#pragma unroll
            for (int r = 0; r < 3; ++r)
                gr[r] = double(L[(3 * r) * N + i]) * g[0] + double(L[(3 * r + 1) * N + i]) * g[1] +
                        double(L[(3 * r + 2) * N + i]) * g[2];
            const double g2 = sq3_rn(gr[0], gr[1], gr[2]);
            const double dens = (1.0 - si) * (1.0 - si) / (4.0 * b.eps0) + b.eps0 * g2;
            acc[2] = b.Gc * (V0i * dens);
        }
    }
    block_sum<3>(acc, part);
}

// measure-plane partials: sum u (3) and sum m0 a (3) over device positions pos[0..m)
template <typename R>
__global__ void __launch_bounds__(kThreads) k_measure(const tl_body b, const int32_t* pos, int64_t m,
                                                       double* part) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (k < m) {
        const int64_t i = pos[k];
        const int64_t N = b.n_all;
        const R* us = static_cast<const R*>(b.us);
        const R* a = static_cast<const R*>(b.a);
        const double m0i = b.uniform ? b.m0c : b.m0[i];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            acc[c] = double(us[4 * i + c]);
            acc[3 + c] = m0i * double(a[c * N + i]);
        }
    }
    block_sum<6>(acc, part);
}

template <typename R, int DIM>
void launch_energies(cudaStream_t st, const tl_body& b, double* part) {
    const unsigned g = tl_blocks(b.n, kThreads);
    if (b.kind == 1) k_energies<R, DIM, 1><<<g, kThreads, 0, st>>>(b, part);
    else k_energies<R, DIM, 2><<<g, kThreads, 0, st>>>(b, part);
}

// VTK snapshot record of every owned particle (output.py:84-127 reads x, u,
// v, the phase field or equivalent plastic strain, and the Cauchy stress of
// constitutive.cauchy_batch): 16 FP64 per particle written at row dst[i] (the
// caller's order), so one contiguous device->host copy delivers the snapshot
// a VTK writer needs.  sigma = sym(F S F^T) / J, zero where J <= J_MIN.
template <typename R>
__global__ void __launch_bounds__(kThreads) k_snapshot(const tl_body b, const int64_t* dst,
                                                       double* out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= b.n) return;
    const int64_t N = b.n_all;
    const R* us = static_cast<const R*>(b.us);
    const R* v = static_cast<const R*>(b.v);
    double* o = out + 16 * dst[i];
    const double u0 = double(us[4 * i]), u1 = double(us[4 * i + 1]), u2 = double(us[4 * i + 2]);
    o[0] = b.Xs[i] + u0;
    o[1] = b.Xs[N + i] + u1;
    o[2] = b.Xs[2 * N + i] + u2;
    o[3] = u0; o[4] = u1; o[5] = u2;
    o[6] = double(v[i]); o[7] = double(v[N + i]); o[8] = double(v[2 * N + i]);
    o[9] = b.model == 3 ? double(static_cast<const R*>(b.epbar)[i]) : double(us[4 * i + 3]);
    const double* F = b.F_out + 9 * i;
    const double* S = b.S_out + 9 * i;
    const double J = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
                     F[2] * (F[3] * F[7] - F[4] * F[6]);
    double sg[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (J > TL_J_MIN) {
        double FS[9], sig[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                FS[3 * r + c] = F[3 * r] * S[c] + F[3 * r + 1] * S[3 + c] + F[3 * r + 2] * S[6 + c];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                sig[3 * r + c] = (FS[3 * r] * F[3 * c] + FS[3 * r + 1] * F[3 * c + 1] +
                                  FS[3 * r + 2] * F[3 * c + 2]) / J;
        sg[0] = sig[0]; sg[1] = sig[4]; sg[2] = sig[8];
        sg[3] = 0.5 * (sig[1] + sig[3]);
        sg[4] = 0.5 * (sig[2] + sig[6]);
        sg[5] = 0.5 * (sig[5] + sig[7]);
    }
    for (int k = 0; k < 6; ++k) o[10 + k] = sg[k];
}

}  // namespace

extern "C" int64_t tl_energy_blocks(int64_t n) { return (int64_t)tl_blocks(n, kThreads); }

extern "C" int tl_energies(tl_stream_t st_, const tl_body* b, double* partials) {
    if (!b || b->n <= 0 || !b->psi_out || !b->v || !b->soff || !b->sidx) {
        tl_set_error("tl_energies: descriptor needs psi_out (host mirrors), v and the neighbour slices");
        return TL_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)st_;
    if (b->precision == 4) {
        if (b->dim == 3) launch_energies<float, 3>(st, *b, partials);
        else launch_energies<float, 2>(st, *b, partials);
    } else {
        if (b->dim == 3) launch_energies<double, 3>(st, *b, partials);
        else launch_energies<double, 2>(st, *b, partials);
    }
    return tl_check_launch("k_energies");
}

extern "C" int tl_measure(tl_stream_t st_, const tl_body* b, const int32_t* pos, int64_t m,
                          double* partials) {
    if (m <= 0) return TL_OK;
    if (!b || !b->a || !b->us) {
        tl_set_error("tl_measure: descriptor needs u|s records and the acceleration planes");
        return TL_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)st_;
    const unsigned g = tl_blocks(m, kThreads);
    if (b->precision == 4) k_measure<float><<<g, kThreads, 0, st>>>(*b, pos, m, partials);
    else k_measure<double><<<g, kThreads, 0, st>>>(*b, pos, m, partials);
    return tl_check_launch("k_measure");
}

extern "C" int tl_snapshot(tl_stream_t st_, const tl_body* b, const int64_t* dst, double* out) {
    if (!b || b->n <= 0 || !b->F_out || !b->S_out || !b->us || !b->v || !dst || !out) {
        tl_set_error("tl_snapshot: descriptor needs the F/S host-layout mirrors, u|s and v");
        return TL_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)st_;
    const unsigned g = tl_blocks(b->n, kThreads);
    if (b->precision == 4) k_snapshot<float><<<g, kThreads, 0, st>>>(*b, dst, out);
    else k_snapshot<double><<<g, kThreads, 0, st>>>(*b, dst, out);
    return tl_check_launch("k_snapshot");
}
