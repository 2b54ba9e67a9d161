// neighbors.cu -- reference-configuration neighbour build on the device.
//
// Replaces kernel_geom.build_pairs / sever_notch_bonds / _csr_from_pairs /
// correction_matrices and the per-pair part of build_adjacency
// (/root/reference/pkg/src/solidsph/kernel_geom.py:65-261).
//
//  1. particles are bucketed into cells of edge >= cutoff (radial 2h, or the
//     nbsrange window) and radix-sorted by cell key (CUB, stable, so each
//     cell lists its particles in ascending original index);
//  2. count / fill passes: one thread per particle i scans the 3^d cells
//     around its own, applies the reference's exact inclusion test to the
//     pair (min(i,j), max(i,j)) -- the orientation scipy's query_pairs hands
//     to the test -- and the notch test to the directed pair i->j, as
//     sever_notch_bonds sees it;
//  3. each row is sorted ascending, giving the lexsort((cols, rows)) order.
// FP64 arithmetic in the tests uses __dmul_rn/__dadd_rn in numpy's evaluation
// order ((dx*dx + dz*dz) + dy*dy, no FMA) so the exact-2h tie-break agrees
// bit for bit.
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "tl_common.cuh"

struct tl_nb_plan {
    cudaStream_t st;
    tl_nb_params p;
    tl_notch* d_notch;
    uint64_t* keys;        // sorted cell keys
    int64_t* order;        // particle index per sorted slot
    int64_t* cell_start;   // dense table (ncell+1) or NULL
    int64_t ncell;
    void* pool;            // one allocation for everything above
};

namespace {

constexpr int kThreads = 256;

struct Grid {
    const double* X;
    int64_t n;
    int mode;
    double cut2, win, lo0, lo1, lo2, cell;
    int64_t d0, d1, d2;
    const uint64_t* keys;
    const int64_t* order;
    const int64_t* cell_start;  // may be NULL -> binary search
    int n_notch;
    const tl_notch* notch;
};

__device__ __forceinline__ int64_t cell_coord(double x, double lo, double cell, int64_t dim) {
    int64_t c = (int64_t)floor((x - lo) / cell);
    return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__global__ void k_cell_keys(int64_t n, const double* __restrict__ X, double lo0, double lo1,
                            double lo2, double cell, int64_t d0, int64_t d1, int64_t d2,
                            uint64_t* __restrict__ keys, int64_t* __restrict__ idx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t c0 = cell_coord(X[3 * i], lo0, cell, d0);
    const int64_t c1 = cell_coord(X[3 * i + 1], lo1, cell, d1);
    const int64_t c2 = cell_coord(X[3 * i + 2], lo2, cell, d2);
    keys[i] = (uint64_t)((c0 * d1 + c1) * d2 + c2);
    idx[i] = i;
}

__global__ void k_cell_start(int64_t n, const uint64_t* __restrict__ keys, int64_t ncell,
                             int64_t* __restrict__ start) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p > n) return;
    // start[c] = first slot with key >= c ; written for the key range ending at p
    const int64_t kcur = p < n ? (int64_t)keys[p] : ncell;
    const int64_t kprev = p > 0 ? (int64_t)keys[p - 1] : -1;
    for (int64_t c = kprev + 1; c <= kcur; ++c) start[c] = p;
}

__device__ __forceinline__ void cell_range(const Grid& g, uint64_t key, int64_t& b, int64_t& e) {
    if (g.cell_start) {
        b = g.cell_start[key];
        e = g.cell_start[key + 1];
        return;
    }
    int64_t lo = 0, hi = g.n;
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (g.keys[m] < key) lo = m + 1; else hi = m;
    }
    b = lo;
    hi = g.n;
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (g.keys[m] <= key) lo = m + 1; else hi = m;
    }
    e = lo;
}

// exact inclusion test on the unordered pair, oriented a < b
__device__ __forceinline__ bool keep_pair(const Grid& g, int64_t a, int64_t b) {
    const double dx = __dsub_rn(g.X[3 * a], g.X[3 * b]);
    const double dy = __dsub_rn(g.X[3 * a + 1], g.X[3 * b + 1]);
    const double dz = __dsub_rn(g.X[3 * a + 2], g.X[3 * b + 2]);
    if (g.mode == 1) return fabs(dx) <= g.win && fabs(dy) <= g.win && fabs(dz) <= g.win;
    double s = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz));
    s = __dadd_rn(s, __dmul_rn(dy, dy));
    return s < g.cut2;
}

__device__ __forceinline__ double dot3rn(double a0, double a1, double a2, const double* b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a0, b[0]), __dmul_rn(a1, b[1])), __dmul_rn(a2, b[2]));
}

// does segment Xa->Xb cross notch q?  (kernel_geom.py:134-159)
__device__ bool crosses(const tl_notch& q, const double* Xa, const double* Xb) {
    const double da = dot3rn(Xa[0] - q.origin[0], Xa[1] - q.origin[1], Xa[2] - q.origin[2], q.nhat);
    const double db = dot3rn(Xb[0] - q.origin[0], Xb[1] - q.origin[1], Xb[2] - q.origin[2], q.nhat);
    const double tol = q.tol_plane;
    const bool opposite = (da < -tol && db > tol) || (da > tol && db < -tol);
    const bool touching = (fabs(da) <= tol && fabs(db) > tol) || (fabs(db) <= tol && fabs(da) > tol);
    if (!(opposite || touching)) return false;
    double den = da - db;
    if (fabs(den) < 1e-300) den = 1e-300;
    double t = da / den;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    double hit[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) hit[a] = Xa[a] + t * (Xb[a] - Xa[a]);
    const double rx = hit[0] - q.origin[0], ry = hit[1] - q.origin[1], rz = hit[2] - q.origin[2];
    const double p0 = dot3rn(rx, ry, rz, q.e1);
    const double p1 = dot3rn(rx, ry, rz, q.e2);
    bool pos = true, neg = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double* A = q.poly[k];
        const double* B = q.poly[(k + 1) & 3];
        const double cr = (B[0] - A[0]) * (p1 - A[1]) - (B[1] - A[1]) * (p0 - A[0]);
        pos = pos && cr >= -q.tol_poly;
        neg = neg && cr <= q.tol_poly;
    }
    return pos || neg;
}

template <bool FILL>
__global__ void k_pairs(Grid g, int64_t* __restrict__ counts, const int64_t* __restrict__ indptr,
                        int32_t* __restrict__ cols) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const double Xi[3] = {g.X[3 * i], g.X[3 * i + 1], g.X[3 * i + 2]};
    const int64_t c0 = cell_coord(Xi[0], g.lo0, g.cell, g.d0);
    const int64_t c1 = cell_coord(Xi[1], g.lo1, g.cell, g.d1);
    const int64_t c2 = cell_coord(Xi[2], g.lo2, g.cell, g.d2);
    int32_t* out = FILL ? cols + indptr[i] : nullptr;
    int64_t cnt = 0;
    for (int64_t a = c0 - 1; a <= c0 + 1; ++a) {
        if (a < 0 || a >= g.d0) continue;
        for (int64_t b = c1 - 1; b <= c1 + 1; ++b) {
            if (b < 0 || b >= g.d1) continue;
            for (int64_t c = c2 - 1; c <= c2 + 1; ++c) {
                if (c < 0 || c >= g.d2) continue;
                int64_t pb, pe;
                cell_range(g, (uint64_t)((a * g.d1 + b) * g.d2 + c), pb, pe);
                for (int64_t p = pb; p < pe; ++p) {
                    const int64_t j = g.order[p];
                    if (j == i) continue;
                    if (!(i < j ? keep_pair(g, i, j) : keep_pair(g, j, i))) continue;
                    bool cut = false;
                    if (g.n_notch) {
                        const double Xj[3] = {g.X[3 * j], g.X[3 * j + 1], g.X[3 * j + 2]};
                        for (int q = 0; q < g.n_notch && !cut; ++q) cut = crosses(g.notch[q], Xi, Xj);
                    }
                    if (cut) continue;
                    if (FILL) out[cnt] = (int32_t)j;
                    ++cnt;
                }
            }
        }
    }
    if (FILL) {
        // rows arrive nearly sorted (cells in x-major order): insertion sort
        for (int64_t k = 1; k < cnt; ++k) {
            const int32_t v = out[k];
            int64_t m = k - 1;
            while (m >= 0 && out[m] > v) {
                out[m + 1] = out[m];
                --m;
            }
            out[m + 1] = v;
        }
    } else {
        counts[i] = cnt;
    }
}

// FP64 kernel factor exactly in the reference's operation order:
// r = sqrt((x^2+y^2)+z^2) (np.linalg.norm), q = r/h, dW/dr = alpha*dw/h,
// grad_base = (dW/dr / r) * r0 (kernel_geom.py:30-62, 236-240).
__device__ __forceinline__ void base_gradient(double dx, double dy, double dz, double h,
                                              double alpha, int kind, double* gb, double* r_out,
                                              double* w_out) {
    const double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    const double q = r / h;
    double w, dw;
    if (kind == 2) {
        const double t = q < 2.0 ? 1.0 - 0.5 * q : 0.0;
        const double t3 = __dmul_rn(__dmul_rn(t, t), t);
        w = __dmul_rn(__dmul_rn(t3, t), __dadd_rn(__dmul_rn(2.0, q), 1.0));
        dw = __dmul_rn(__dmul_rn(-5.0, q), t3);
    } else {
        const double tm = 2.0 - q;
        if (q < 1.0) {
            w = 1.0 - 1.5 * q * q + 0.75 * q * q * q;
            dw = -3.0 * q + 2.25 * q * q;
        } else if (q < 2.0) {
            w = 0.25 * tm * tm * tm;
            dw = -0.75 * tm * tm;
        } else {
            w = 0.0;
            dw = 0.0;
        }
    }
    const double dwdr = alpha * dw / h;
    const double f = r == 0.0 ? 0.0 : dwdr / r;
    gb[0] = __dmul_rn(f, dx);
    gb[1] = __dmul_rn(f, dy);
    gb[2] = __dmul_rn(f, dz);
    if (r == 0.0) gb[0] = gb[1] = gb[2] = 0.0;
    if (r_out) *r_out = r;
    if (w_out) *w_out = alpha * w;
}

// sigma_max of a 3x3 from the largest eigenvalue of its Gram matrix
__device__ double smax3(const double* A) {
    double G[9], w[3], Q[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            G[3 * r + c] = A[r] * A[c] + A[3 + r] * A[3 + c] + A[6 + r] * A[6 + c];
    tl::eig3_jacobi(G, w, Q, 1e-30);
    return sqrt(fmax(w[0], 0.0));
}

__global__ void k_correction(int64_t n, const int64_t* __restrict__ indptr,
                             const int32_t* __restrict__ indices, const double* __restrict__ X,
                             const double* __restrict__ V0, double h, double alpha, int kind,
                             int dim, int correction, double* __restrict__ L, int64_t* fallbacks) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int fb = 0;
    if (i < n) {
        double* Li = L + 9 * i;
        if (!correction) {
#pragma unroll
            for (int q = 0; q < 9; ++q) Li[q] = (q % 4 == 0) ? 1.0 : 0.0;
        } else {
            double A[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            const double xi = X[3 * i], yi = X[3 * i + 1], zi = X[3 * i + 2];
            for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
                const int64_t j = indices[k];
                const double dx = __dsub_rn(xi, X[3 * j]), dy = __dsub_rn(yi, X[3 * j + 1]),
                             dz = __dsub_rn(zi, X[3 * j + 2]);
                double gb[3];
                base_gradient(dx, dy, dz, h, alpha, kind, gb, nullptr, nullptr);
                const double d[3] = {__dsub_rn(X[3 * j], xi), __dsub_rn(X[3 * j + 1], yi),
                                     __dsub_rn(X[3 * j + 2], zi)};
                const double vj = V0[j];
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    const double vg = __dmul_rn(vj, gb[r]);
#pragma unroll
                    for (int c = 0; c < 3; ++c) A[3 * r + c] = __dadd_rn(A[3 * r + c], __dmul_rn(vg, d[c]));
                }
            }
            if (dim == 2) {
                A[3] = A[4] = A[5] = 0.0;
                A[1] = A[7] = 0.0;
                A[4] = 1.0;
            }
            bool finite = true;
#pragma unroll
            for (int q = 0; q < 9; ++q) finite = finite && isfinite(A[q]);
            double Ai[9];
            double cond = INFINITY;
            if (finite && tl::det3(A) != 0.0) {
                tl::inv3(A, Ai);
                cond = smax3(A) * smax3(Ai);
                if (!isfinite(cond)) cond = INFINITY;
            }
            if (finite && cond < 1.0e8) {
#pragma unroll
                for (int q = 0; q < 9; ++q) Li[q] = Ai[q];
            } else {
#pragma unroll
                for (int q = 0; q < 9; ++q) Li[q] = (q % 4 == 0) ? 1.0 : 0.0;
                fb = 1;
            }
        }
    }
    int t = tl::warp_sum_int(fb);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd((unsigned long long*)fallbacks, (unsigned long long)t);
}

__device__ __forceinline__ void matvec_rn(const double* L, const double* g, double* o) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
        o[a] = __dadd_rn(__dadd_rn(__dmul_rn(L[3 * a], g[0]), __dmul_rn(L[3 * a + 1], g[1])),
                         __dmul_rn(L[3 * a + 2], g[2]));
}

__global__ void k_expand(int64_t n, const int64_t* __restrict__ indptr,
                         const int32_t* __restrict__ indices, const double* __restrict__ X,
                         const double* __restrict__ L, double h, double alpha, int kind,
                         int64_t* rows, double* r0, double* r0norm, double* w0, double* grad0,
                         double* grad0r) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double xi = X[3 * i], yi = X[3 * i + 1], zi = X[3 * i + 2];
    double Li[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) Li[q] = L[9 * i + q];
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
        const int64_t j = indices[k];
        const double dx = __dsub_rn(xi, X[3 * j]), dy = __dsub_rn(yi, X[3 * j + 1]),
                     dz = __dsub_rn(zi, X[3 * j + 2]);
        double gb[3], r, w;
        base_gradient(dx, dy, dz, h, alpha, kind, gb, &r, &w);
        if (rows) rows[k] = i;
        if (r0) {
            r0[3 * k] = dx;
            r0[3 * k + 1] = dy;
            r0[3 * k + 2] = dz;
        }
        if (r0norm) r0norm[k] = r;
        if (w0) w0[k] = w;
        double g[3];
        if (grad0) {
            matvec_rn(Li, gb, g);
            grad0[3 * k] = g[0];
            grad0[3 * k + 1] = g[1];
            grad0[3 * k + 2] = g[2];
        }
        if (grad0r) {
            double Lj[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) Lj[q] = L[9 * j + q];
            const double mg[3] = {-gb[0], -gb[1], -gb[2]};
            matvec_rn(Lj, mg, g);
            grad0r[3 * k] = g[0];
            grad0r[3 * k + 1] = g[1];
            grad0r[3 * k + 2] = g[2];
        }
    }
}

__global__ void k_sell_len(int64_t n, const int64_t* __restrict__ indptr, int32_t* slen) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nw = (n + 31) / 32;
    if ((i >> 5) >= nw) return;
    int len = i < n ? (int)(indptr[i + 1] - indptr[i]) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    // slices are a whole number of TL_SELL_GROUP slots so the step kernels
    // gather neighbours in unconditional groups
    if ((threadIdx.x & 31) == 0) slen[i >> 5] = (len + TL_SELL_GROUP - 1) / TL_SELL_GROUP * TL_SELL_GROUP;
}

__global__ void k_sell_fill(int64_t n, const int64_t* __restrict__ indptr,
                            const int32_t* __restrict__ indices, const int64_t* __restrict__ soff,
                            int32_t* __restrict__ sidx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nw = (n + 31) / 32;
    const int64_t w = i >> 5;
    if (w >= nw) return;
    const int lane = (int)(i & 31);
    const int64_t base = soff[w];
    const int64_t slots = (soff[w + 1] - base) / 32;
    const int64_t b = i < n ? indptr[i] : 0;
    const int64_t len = i < n ? indptr[i + 1] - b : 0;
    // padding points at the particle itself: r0 = 0 makes every pair term
    // vanish exactly, so the step kernels need no per-lane bounds test
    const int32_t self = i < n ? (int32_t)i : 0;
    for (int64_t k = 0; k < slots; ++k) sidx[base + 32 * k + lane] = k < len ? indices[b + k] : self;
}

}  // namespace

extern "C" int tl_nb_plan_create(tl_stream_t st_, const tl_nb_params* p, tl_nb_plan** out) {
    if (!p || !out || p->n < 2 || !p->X) {
        tl_set_error("tl_nb_plan_create: bad arguments");
        return TL_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)st_;
    tl_nb_plan* plan = new tl_nb_plan();
    plan->st = st;
    plan->p = *p;
    const int64_t n = p->n;
    const int64_t ncell = p->dims[0] * p->dims[1] * p->dims[2];
    plan->ncell = ncell;
    const bool dense = ncell <= 8 * n + (1 << 20);
    int end_bit = 1;
    while (end_bit < 64 && (uint64_t(1) << end_bit) < (uint64_t)ncell) ++end_bit;
    // temp storage size for the radix sort
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (int64_t*)nullptr, (int64_t*)nullptr, n, 0, end_bit, st);
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t nn = sizeof(uint64_t) * (size_t)n;
    size_t bytes = al(nn) * 2 + al(sizeof(int64_t) * n) * 2 + al(sort_bytes) +
                   (dense ? al(sizeof(int64_t) * (ncell + 1)) : 0) +
                   al(sizeof(tl_notch) * (p->n_notch > 0 ? p->n_notch : 1));
    char* pool = nullptr;
    TL_TRY_CUDA(cudaMallocAsync((void**)&pool, bytes, st));
    plan->pool = pool;
    char* cur = pool;
    auto take = [&](size_t b) { char* r = cur; cur += al(b); return r; };
    uint64_t* keys_in = (uint64_t*)take(nn);
    plan->keys = (uint64_t*)take(nn);
    int64_t* idx_in = (int64_t*)take(sizeof(int64_t) * n);
    plan->order = (int64_t*)take(sizeof(int64_t) * n);
    void* sort_tmp = take(sort_bytes);
    plan->cell_start = dense ? (int64_t*)take(sizeof(int64_t) * (ncell + 1)) : nullptr;
    plan->d_notch = (tl_notch*)take(sizeof(tl_notch) * (p->n_notch > 0 ? p->n_notch : 1));
    if (p->n_notch > 0)
        TL_TRY_CUDA(cudaMemcpyAsync(plan->d_notch, p->notches, sizeof(tl_notch) * p->n_notch,
                                    cudaMemcpyHostToDevice, st));
    k_cell_keys<<<tl_blocks(n, kThreads), kThreads, 0, st>>>(
        n, p->X, p->lo[0], p->lo[1], p->lo[2], p->cell, p->dims[0], p->dims[1], p->dims[2],
        keys_in, idx_in);
    int rc = tl_check_launch("k_cell_keys");
    if (rc) return rc;
    TL_TRY_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, keys_in, plan->keys, idx_in,
                                                plan->order, n, 0, end_bit, st));
    if (dense) {
        k_cell_start<<<tl_blocks(n + 1, kThreads), kThreads, 0, st>>>(n, plan->keys, ncell,
                                                                     plan->cell_start);
        rc = tl_check_launch("k_cell_start");
        if (rc) return rc;
    }
    *out = plan;
    return TL_OK;
}

static Grid make_grid(const tl_nb_plan* plan) {
    const tl_nb_params& p = plan->p;
    Grid g;
    g.X = p.X;
    g.n = p.n;
    g.mode = p.mode;
    g.cut2 = (2.0 * p.h) * (2.0 * p.h);
    g.win = p.win;
    g.lo0 = p.lo[0];
    g.lo1 = p.lo[1];
    g.lo2 = p.lo[2];
    g.cell = p.cell;
    g.d0 = p.dims[0];
    g.d1 = p.dims[1];
    g.d2 = p.dims[2];
    g.keys = plan->keys;
    g.order = plan->order;
    g.cell_start = plan->cell_start;
    g.n_notch = p.n_notch;
    g.notch = plan->d_notch;
    return g;
}

extern "C" int tl_nb_count(tl_nb_plan* plan, int64_t* counts) {
    Grid g = make_grid(plan);
    k_pairs<false><<<tl_blocks(g.n, kThreads), kThreads, 0, plan->st>>>(g, counts, nullptr, nullptr);
    return tl_check_launch("k_pairs<count>");
}

extern "C" int tl_nb_fill(tl_nb_plan* plan, const int64_t* indptr, int32_t* indices) {
    Grid g = make_grid(plan);
    k_pairs<true><<<tl_blocks(g.n, kThreads), kThreads, 0, plan->st>>>(g, nullptr, indptr, indices);
    return tl_check_launch("k_pairs<fill>");
}

extern "C" int tl_nb_plan_destroy(tl_nb_plan* plan) {
    if (!plan) return TL_OK;
    cudaError_t e = cudaFreeAsync(plan->pool, plan->st);
    delete plan;
    if (e != cudaSuccess) {
        tl_set_error("cudaFreeAsync: %s", cudaGetErrorString(e));
        return TL_ERR_CUDA;
    }
    return TL_OK;
}

extern "C" int tl_correction(tl_stream_t st, int64_t n, const int64_t* indptr,
                             const int32_t* indices, const double* X, const double* V0, double h,
                             double alpha, int kind, int dim, int correction, double* L,
                             int64_t* fallbacks) {
    if (n <= 0) return TL_OK;
    k_correction<<<tl_blocks(n, kThreads), kThreads, 0, (cudaStream_t)st>>>(
        n, indptr, indices, X, V0, h, alpha, kind, dim, correction, L, fallbacks);
    return tl_check_launch("k_correction");
}

extern "C" int tl_adjacency_expand(tl_stream_t st, int64_t n, const int64_t* indptr,
                                   const int32_t* indices, const double* X, const double* L,
                                   double h, double alpha, int kind, int64_t* rows, double* r0,
                                   double* r0norm, double* w0, double* grad0, double* grad0r) {
    if (n <= 0) return TL_OK;
    k_expand<<<tl_blocks(n, kThreads), kThreads, 0, (cudaStream_t)st>>>(
        n, indptr, indices, X, L, h, alpha, kind, rows, r0, r0norm, w0, grad0, grad0r);
    return tl_check_launch("k_expand");
}

extern "C" int tl_sell_lengths(tl_stream_t st, int64_t n, const int64_t* indptr, int32_t* slen) {
    if (n <= 0) return TL_OK;
    const int64_t nt = ((n + 31) / 32) * 32;
    k_sell_len<<<tl_blocks(nt, kThreads), kThreads, 0, (cudaStream_t)st>>>(n, indptr, slen);
    return tl_check_launch("k_sell_len");
}

extern "C" int tl_sell_fill(tl_stream_t st, int64_t n, const int64_t* indptr,
                            const int32_t* indices, const int64_t* soff, int32_t* sidx) {
    if (n <= 0) return TL_OK;
    const int64_t nt = ((n + 31) / 32) * 32;
    k_sell_fill<<<tl_blocks(nt, kThreads), kThreads, 0, (cudaStream_t)st>>>(n, indptr, indices,
                                                                          soff, sidx);
    return tl_check_launch("k_sell_fill");
}
