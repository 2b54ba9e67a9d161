// tl_common.cuh -- shared device helpers for libtlsph (sm_100a).
//
// 3x3 tensors are row-major Real[9].  Real is float (FP32 mode) or double
// (FP64 mode); reference-configuration geometry (positions, neighbour
// tests, correction matrices) is always FP64.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/tlsph.h"

#define TL_J_MIN 1.0e-6   // reference core.py:45

namespace tl {

template <typename R> struct Vec4;
template <> struct Vec4<float> { using T = float4; };
template <> struct Vec4<double> { using T = double4; };

template <typename R>
__device__ __forceinline__ typename Vec4<R>::T ld4(const R* p) {
    return *reinterpret_cast<const typename Vec4<R>::T*>(p);
}
template <typename R>
__device__ __forceinline__ void st4(R* p, R a, R b, R c, R d) {
    typename Vec4<R>::T v;
    v.x = a; v.y = b; v.z = c; v.w = d;
    *reinterpret_cast<typename Vec4<R>::T*>(p) = v;
}
// read-only-path variants (one LDG.128 per float4, two per double4)
__device__ __forceinline__ float4 ldg4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ double4 ldg4(const double* p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

template <typename T>
__device__ __forceinline__ T det3(const T* A) {
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
           A[2] * (A[3] * A[7] - A[4] * A[6]);
}

// cofactor inverse; returns det (callers decide what a tiny det means)
template <typename T>
__device__ __forceinline__ T inv3(const T* A, T* R) {
    T d = det3(A);
    T id = T(1) / d;
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

template <typename T>
__device__ __forceinline__ void mm3(const T* A, const T* B, T* C) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            C[3 * r + c] = A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c] + A[3 * r + 2] * B[6 + c];
}

// C = A * B^T
template <typename T>
__device__ __forceinline__ void mmT3(const T* A, const T* B, T* C) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            C[3 * r + c] = A[3 * r] * B[3 * c] + A[3 * r + 1] * B[3 * c + 1] + A[3 * r + 2] * B[3 * c + 2];
}

// cyclic Jacobi, symmetric 3x3, eigenvalues descending, eigenvectors in Q's
// columns; returns sweeps (64 = not converged).  Same rotation sequence as the
// reference solver (backends/fast.py:45-108); tol_rel scales the stopping
// test (1e-30 in FP64 as in the reference; FP32 needs a representable one).
template <typename T>
__device__ __forceinline__ int eig3_jacobi(const T* Ain, T* w, T* Q, T tol_rel) {
    T a[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) a[3 * r + c] = T(0.5) * (Ain[3 * r + c] + Ain[3 * c + r]);
#pragma unroll
    for (int k = 0; k < 9; ++k) Q[k] = (k % 4 == 0) ? T(1) : T(0);
    T scale = T(0);
#pragma unroll
    for (int k = 0; k < 9; ++k) scale = fmax(scale, fabs(a[k]));
    if (scale == T(0)) {
        w[0] = w[1] = w[2] = T(0);
        return 0;
    }
    const T tol = tol_rel * scale * scale;
    const T tiny = sizeof(T) == 8 ? T(1e-300) : T(1e-37);
    int sweeps = 0;
    while (sweeps < 64) {
        T off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
        if (off <= tol) break;
#pragma unroll
        for (int pq = 0; pq < 3; ++pq) {
            const int p = pq == 2 ? 1 : 0;
            const int q = pq == 0 ? 1 : 2;
            T apq = a[3 * p + q];
            if (fabs(apq) < tiny) continue;
            T theta = T(0.5) * (a[3 * q + q] - a[3 * p + p]) / apq;
            T t = theta >= T(0) ? T(1) / (theta + sqrt(theta * theta + T(1)))
                                : T(-1) / (-theta + sqrt(theta * theta + T(1)));
            T c = T(1) / sqrt(t * t + T(1));
            T s = t * c;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                T x = a[3 * k + p], y = a[3 * k + q];
                a[3 * k + p] = c * x - s * y;
                a[3 * k + q] = s * x + c * y;
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                T x = a[3 * p + k], y = a[3 * q + k];
                a[3 * p + k] = c * x - s * y;
                a[3 * q + k] = s * x + c * y;
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                T x = Q[3 * k + p], y = Q[3 * k + q];
                Q[3 * k + p] = c * x - s * y;
                Q[3 * k + q] = s * x + c * y;
            }
        }
        ++sweeps;
    }
    w[0] = a[0];
    w[1] = a[4];
    w[2] = a[8];
    // selection sort, descending, swapping eigenvector columns
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        int m = i;
#pragma unroll
        for (int j = i + 1; j < 3; ++j)
            if (w[j] > w[m]) m = j;
        if (m != i) {
            T tmp = w[i]; w[i] = w[m]; w[m] = tmp;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                tmp = Q[3 * k + i]; Q[3 * k + i] = Q[3 * k + m]; Q[3 * k + m] = tmp;
            }
        }
    }
    return sweeps;
}

// radial kernel factor: grad_base = fac * r0 with fac = (dW/dr)/r, written
// with rs = 1/r (0 at r = 0, so coincident pairs and the self-padding of the
// sliced ELL contribute exactly nothing).  KIND 1 = cubic spline, 2 =
// Wendland C2 (reference kernel_geom.py:30-62); a_ih = alpha / h.
__device__ __forceinline__ float rsqrt_pos(float x) { return x > 0.f ? rsqrtf(x) : 0.f; }
__device__ __forceinline__ double rsqrt_pos(double x) { return x > 0.0 ? rsqrt(x) : 0.0; }
// --- asynchronous copies (TMA bulk, LDGSTS) and mbarriers, inline PTX ------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "TL_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra TL_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// TMA 1D bulk copy global -> shared, completion counted on `bar` (16-byte
// aligned addresses, bytes a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 16-byte LDGSTS (L2 only)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// TMA bulk prefetch of [p, p + bytes) into L2 (rounded out to 16 bytes)
__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
    const uintptr_t a = (uintptr_t)p & ~uintptr_t(15);
    const uintptr_t e = ((uintptr_t)p + bytes + 15) & ~uintptr_t(15);
    if (e > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a))
                     : "memory");
}

// 1/sqrt(max(x, smallest normal)): finite for x = 0 (self-padding pairs)
__device__ __forceinline__ float rsqrt_floor(float x) { return rsqrtf(fmaxf(x, 1.17549435e-38f)); }
__device__ __forceinline__ double rsqrt_floor(double x) { return rsqrt(fmax(x, 2.2250738585072014e-308)); }

template <typename T, int KIND>
__device__ __forceinline__ T kernel_fac(T r2, T rs, T inv_h, T a_ih) {
    const T q = r2 * rs * inv_h;
    T dw;
    if (KIND == 2) {
        const T t = q < T(2) ? T(1) - T(0.5) * q : T(0);
        dw = T(-5) * q * t * t * t;
    } else {
        const T tm = T(2) - q;
        dw = q < T(1) ? T(-3) * q + T(2.25) * q * q : (q < T(2) ? T(-0.75) * tm * tm : T(0));
    }
    return a_ih * dw * rs;
}

// a + b*c with both roundings (no FMA contraction): the integrator updates
// follow numpy's `x += dt * y` rounding exactly
__device__ __forceinline__ double axpy_rn(double a, double b, double c) {
    return __dadd_rn(a, __dmul_rn(b, c));
}
__device__ __forceinline__ float axpy_rn(float a, float b, float c) {
    return __fadd_rn(a, __fmul_rn(b, c));
}
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// atomic max for non-negative doubles via their IEEE bit patterns
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* addr, double v) {
    atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, (long long)__shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Programmatic dependent launch: the step kernels (clock, passes, predictor)
// are launched with programmatic stream serialisation (tl_launch), so a
// kernel's CTAs are scheduled while its predecessor drains and its launch
// latency overlaps the predecessor's tail.  Every such kernel first waits for
// the predecessor grid to complete and flush its memory (griddepcontrol.wait,
// a no-op for a normal launch), then lets its own dependents launch.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace tl

// launch with programmatic stream serialisation (TLSPH_PDL=0: plain launch);
// only for kernels that call tl::pdl_enter() before touching global memory
bool tl_pdl_enabled();
template <typename... P, typename... A>
cudaError_t tl_launch(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      A&&... args) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = tl_pdl_enabled() ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<A&&>(args)...);
}

// error plumbing for the C ABI: every entry point returns 0 or a negative
// code; the message is kept per thread and read with tl_last_error().
void tl_set_error(const char* fmt, ...);
int tl_check_launch(const char* what);

#define TL_TRY_CUDA(expr)                                                       \
    do {                                                                        \
        cudaError_t e_ = (expr);                                                \
        if (e_ != cudaSuccess) {                                                \
            tl_set_error("%s failed: %s", #expr, cudaGetErrorString(e_));       \
            return TL_ERR_CUDA;                                                 \
        }                                                                       \
    } while (0)

static inline unsigned tl_blocks(long long n, int threads) {
    return (unsigned)((n + threads - 1) / threads);
}
