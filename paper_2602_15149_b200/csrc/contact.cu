// contact.cu -- penalty contact between bodies on the device (SURVEY.md 8(f)
// rank 3; dynamics.py:81-135 + backends/fast.py:426-469).
//
// The reference's only per-step Eulerian search: cross-body particle pairs
// closer than dp_contact = (dp_a + dp_b)/2 in the CURRENT configuration
// x = X + u get a normal spring-dashpot force plus a Coulomb-capped
// tangential force, equal and opposite.  It finds pairs with a cKDTree on the
// AABB-overlap gate and accumulates them sequentially in (i of a ascending,
// j of b ascending) order.
//
// Here, per body pair: a cell grid over the gate (cells >= dp_contact), built
// from both bodies' current positions; then one gather kernel per side.  A
// particle of body a collects its partners in b (<= TL_CONTACT_CAP), sorts
// them by original index and accumulates f/m_a in that order; a particle of
// b does the same over its partners in a with the force evaluated in the
// (i of a, j of b) orientation and subtracted -- exactly the reference's
// per-particle summation order, with no atomics on the accumulators.  The
// gate never drops a pair closer than dp_contact, so the result equals the
// reference's global search.  Everything stays on the device: no host sync.
#include <cub/cub.cuh>

#include "tl_common.cuh"

namespace {

constexpr int kThreads = 256;

struct Grid {
    double lo[3];
    double inv_cell;
    int32_t dims[3];
    int32_t active;   // gate non-empty
    int64_t ncell;
};

__device__ __forceinline__ double xcomp(const tl_contact_side& s, int c, int64_t i) {
    const double u = s.precision == 4 ? double(static_cast<const float*>(s.us)[4 * i + c])
                                      : static_cast<const double*>(s.us)[4 * i + c];
    return s.Xs[c * s.n_all + i] + u;
}

__device__ __forceinline__ double vcomp(const tl_contact_side& s, int c, int64_t i) {
    return s.precision == 4 ? double(static_cast<const float*>(s.v)[c * s.n_all + i])
                            : static_cast<const double*>(s.v)[c * s.n_all + i];
}

// ordered-int encoding of doubles for atomicMin/Max
__device__ __forceinline__ long long ord(double x) {
    long long b = __double_as_longlong(x);
    return b >= 0 ? b : b ^ 0x7fffffffffffffffLL;
}
__device__ __forceinline__ double unord(long long b) {
    return __longlong_as_double(b >= 0 ? b : b ^ 0x7fffffffffffffffLL);
}

// bbox[0..2] = ord(min x), bbox[3..5] = ord(max x) of a body's current positions
__global__ void k_bbox(const tl_contact_side s, long long* bbox) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    if (i < s.n) {
#pragma unroll
        for (int c = 0; c < 3; ++c) lo[c] = hi[c] = xcomp(s, c, i);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
            hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
        }
    }
    if ((threadIdx.x & 31) == 0 && lo[0] <= hi[0]) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            atomicMin(&bbox[c], ord(lo[c]));
            atomicMax(&bbox[3 + c], ord(hi[c]));
        }
    }
}

__global__ void k_bbox_init(long long* bbox) {
    if (threadIdx.x < 3) {
        bbox[threadIdx.x] = ord(INFINITY);
        bbox[3 + threadIdx.x] = ord(-INFINITY);
    }
}

// gate = overlap of the two boxes inflated by dpc (dynamics.py:100-105);
// cells of at least dpc, coarsened until the grid fits `cap` cells
__global__ void k_grid(const long long* ba, const long long* bb, double dpc, int dim, int64_t cap,
                       Grid* g) {
    double lo[3], hi[3];
    int active = 1;
    for (int c = 0; c < 3; ++c) {
        lo[c] = fmax(unord(ba[c]), unord(bb[c])) - dpc;
        hi[c] = fmin(unord(ba[3 + c]), unord(bb[3 + c])) + dpc;
        if (lo[c] > hi[c]) active = 0;
    }
    double cell = dpc;
    int32_t dims[3];
    int64_t ncell = 1;
    for (int it = 0; it < 64; ++it) {
        ncell = 1;
        for (int c = 0; c < 3; ++c) {
            const double ext = active ? hi[c] - lo[c] : 0.0;
            dims[c] = (dim == 2 && c == 1) ? 1 : (int32_t)floor(ext / cell) + 1;
            ncell *= dims[c];
        }
        if (ncell <= cap) break;
        cell *= 1.5;
    }
    for (int c = 0; c < 3; ++c) {
        g->lo[c] = lo[c];
        g->dims[c] = dims[c];
    }
    g->inv_cell = 1.0 / cell;
    g->active = active;
    g->ncell = active ? ncell : 0;
}

// inside the grid (a superset of the gate: partners lie in the gate)
__device__ __forceinline__ bool in_gate(const Grid& g, const double* x, int dim) {
    for (int c = 0; c < 3; ++c) {
        if (dim == 2 && c == 1) continue;
        const double hi = g.lo[c] + g.dims[c] / g.inv_cell;
        if (x[c] < g.lo[c] || x[c] > hi) return false;
    }
    return true;
}

__device__ __forceinline__ int cell_coord(const Grid& g, int c, double x) {
    int k = (int)floor((x - g.lo[c]) * g.inv_cell);
    return min(max(k, 0), g.dims[c] - 1);
}

__device__ __forceinline__ int64_t cell_of(const Grid& g, const double* x, int dim) {
    const int cx = cell_coord(g, 0, x[0]);
    const int cy = dim == 3 ? cell_coord(g, 1, x[1]) : 0;
    const int cz = cell_coord(g, 2, x[2]);
    return ((int64_t)cz * g.dims[1] + cy) * g.dims[0] + cx;
}

// per-cell counts of a side's particles inside the gate
__global__ void k_cell_count(const tl_contact_side s, const Grid* gp, int dim, int32_t* cnt,
                             int32_t* cellid) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    const Grid g = *gp;
    int32_t id = -1;
    if (g.active) {
        const double x[3] = {xcomp(s, 0, i), xcomp(s, 1, i), xcomp(s, 2, i)};
        if (in_gate(g, x, dim)) {
            id = (int32_t)cell_of(g, x, dim);
            atomicAdd(&cnt[id], 1);
        }
    }
    cellid[i] = id;
}

__global__ void k_cell_fill(const tl_contact_side s, const int32_t* cellid, const int32_t* start,
                            int32_t* cursor, int32_t* items) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    const int32_t id = cellid[i];
    if (id < 0) return;
    items[start[id] + atomicAdd(&cursor[id], 1)] = (int32_t)i;
}

struct PairParams {
    double dpc, k_n, c_n, kfric;
};

// force on particle ia of body A from jb of body B (fast.py:434-469 order)
__device__ __forceinline__ void pair_force(const tl_contact_side& A, int64_t ia,
                                           const tl_contact_side& B, int64_t jb, const PairParams& p,
                                           double f[3], bool& touch, bool& warn) {
    const double d0 = xcomp(A, 0, ia) - xcomp(B, 0, jb);
    const double d1 = xcomp(A, 1, ia) - xcomp(B, 1, jb);
    const double d2 = xcomp(A, 2, ia) - xcomp(B, 2, jb);
    double dist = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    touch = dist < p.dpc;
    warn = false;
    f[0] = f[1] = f[2] = 0.0;
    if (!touch) return;
    double n0, n1, n2;
    if (dist < 1e-12) {
        n0 = 1.0; n1 = 0.0; n2 = 0.0;
        dist = 1e-12;
        warn = true;
    } else {
        n0 = d0 / dist; n1 = d1 / dist; n2 = d2 / dist;
    }
    const double overlap = p.dpc - dist;
    const double dv0 = vcomp(A, 0, ia) - vcomp(B, 0, jb);
    const double dv1 = vcomp(A, 1, ia) - vcomp(B, 1, jb);
    const double dv2 = vcomp(A, 2, ia) - vcomp(B, 2, jb);
    const double vn = dv0 * n0 + dv1 * n1 + dv2 * n2;
    double fn = p.k_n * overlap - p.c_n * vn;
    if (fn < 0.0) fn = 0.0;
    f[0] = fn * n0; f[1] = fn * n1; f[2] = fn * n2;
    if (p.kfric > 0.0) {
        const double t0 = dv0 - vn * n0, t1 = dv1 - vn * n1, t2 = dv2 - vn * n2;
        const double vtn = sqrt(t0 * t0 + t1 * t1 + t2 * t2);
        if (vtn > 1e-14) {
            f[0] -= p.kfric * fn * t0 / vtn;
            f[1] -= p.kfric * fn * t1 / vtn;
            f[2] -= p.kfric * fn * t2 / vtn;
        }
    }
}

#ifndef TL_CONTACT_CAP
#define TL_CONTACT_CAP 64
#endif

// Gather for the particles of side S (its partners on side O, found through
// O's cell lists).  S_IS_A: S plays the reference's body a (force += f/m),
// else body b (force -= f(a=O, b=S)/m).  Partners are applied in ascending
// original index of O.
template <bool S_IS_A>
__global__ void __launch_bounds__(kThreads) k_contact_gather(
    const tl_contact_side S, const tl_contact_side O, const Grid* gp, int dim,
    const int32_t* ostart, const int32_t* ocnt, const int32_t* oitems, PairParams p,
    double* acc /* 3 planes, stride S.n_all */, unsigned long long* warn_count,
    unsigned long long* overflow) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= S.n) return;
    const Grid g = *gp;
    if (!g.active) return;
    const double x[3] = {xcomp(S, 0, i), xcomp(S, 1, i), xcomp(S, 2, i)};
    if (!in_gate(g, x, dim)) return;
    // partners lie within dpc <= cell of x, i.e. in the neighbouring cells
    int32_t cand[TL_CONTACT_CAP];
    int32_t key[TL_CONTACT_CAP];
    int nc = 0;
    const int cx = cell_coord(g, 0, x[0]), cz = cell_coord(g, 2, x[2]);
    const int cy = dim == 3 ? cell_coord(g, 1, x[1]) : 0;
    const int ylo = dim == 3 ? max(cy - 1, 0) : 0, yhi = dim == 3 ? min(cy + 1, g.dims[1] - 1) : 0;
    for (int zz = max(cz - 1, 0); zz <= min(cz + 1, g.dims[2] - 1); ++zz)
        for (int yy = ylo; yy <= yhi; ++yy)
            for (int xx = max(cx - 1, 0); xx <= min(cx + 1, g.dims[0] - 1); ++xx) {
                const int64_t c = ((int64_t)zz * g.dims[1] + yy) * g.dims[0] + xx;
                for (int32_t k = ostart[c]; k < ostart[c] + ocnt[c]; ++k) {
                    const int32_t j = oitems[k];
                    const double d0 = x[0] - xcomp(O, 0, j), d1 = x[1] - xcomp(O, 1, j),
                                 d2 = x[2] - xcomp(O, 2, j);
                    if (d0 * d0 + d1 * d1 + d2 * d2 >= 1.0000001 * p.dpc * p.dpc) continue;
                    if (nc == TL_CONTACT_CAP) {
                        atomicAdd(overflow, 1ull);
                        continue;
                    }
                    cand[nc] = j;
                    key[nc] = O.perm ? O.perm[j] : j;
                    ++nc;
                }
            }
    if (nc == 0) return;
    // insertion sort by original index
    for (int a = 1; a < nc; ++a) {
        const int32_t kj = key[a], cj = cand[a];
        int b = a - 1;
        while (b >= 0 && key[b] > kj) {
            key[b + 1] = key[b];
            cand[b + 1] = cand[b];
            --b;
        }
        key[b + 1] = kj;
        cand[b + 1] = cj;
    }
    const double mi = S.uniform ? S.m0c : S.m0[i];
    double a0 = acc[i], a1 = acc[S.n_all + i], a2 = acc[2 * S.n_all + i];
    for (int q = 0; q < nc; ++q) {
        double f[3];
        bool touch, warn;
        if (S_IS_A) pair_force(S, i, O, cand[q], p, f, touch, warn);
        else pair_force(O, cand[q], S, i, p, f, touch, warn);
        if (!touch) continue;
        if (S_IS_A) {
            if (warn) atomicAdd(warn_count, 1ull);
            a0 += f[0] / mi; a1 += f[1] / mi; a2 += f[2] / mi;
        } else {
            a0 -= f[0] / mi; a1 -= f[1] / mi; a2 -= f[2] / mi;
        }
    }
    acc[i] = a0;
    acc[S.n_all + i] = a1;
    acc[2 * S.n_all + i] = a2;
}

}  // namespace

extern "C" int tl_contact_workspace_bytes(int64_t n_a, int64_t n_b, int64_t cell_cap,
                                          int64_t* bytes) {
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (int32_t*)nullptr, (int32_t*)nullptr, (int)cell_cap);
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    *bytes = (int64_t)(al(sizeof(Grid)) + 2 * al(6 * sizeof(long long)) +
                       2 * 3 * al((size_t)cell_cap * 4) + al((size_t)n_a * 4) + al((size_t)n_b * 4) +
                       al((size_t)n_a * 4) + al((size_t)n_b * 4) + al(scan) + 256);
    return TL_OK;
}

extern "C" int tl_contact_pair(tl_stream_t st_, const tl_contact_side* a, const tl_contact_side* b,
                               int dim, double dpc, double k_n, double c_n, double kfric,
                               int64_t cell_cap, void* work, int64_t work_bytes, double* acc_a,
                               double* acc_b, unsigned long long* counters) {
    cudaStream_t st = (cudaStream_t)st_;
    int64_t need = 0;
    tl_contact_workspace_bytes(a->n, b->n, cell_cap, &need);
    if (work_bytes < need) {
        tl_set_error("tl_contact_pair: workspace of %lld bytes, need %lld", (long long)work_bytes,
                     (long long)need);
        return TL_ERR_ARG;
    }
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    char* w = (char*)work;
    Grid* g = (Grid*)w; w += al(sizeof(Grid));
    long long* bba = (long long*)w; w += al(6 * sizeof(long long));
    long long* bbb = (long long*)w; w += al(6 * sizeof(long long));
    int32_t* cnt[2]; int32_t* start[2]; int32_t* cur[2]; int32_t* cid[2]; int32_t* items[2];
    for (int k = 0; k < 2; ++k) {
        cnt[k] = (int32_t*)w; w += al((size_t)cell_cap * 4);
        start[k] = (int32_t*)w; w += al((size_t)cell_cap * 4);
        cur[k] = (int32_t*)w; w += al((size_t)cell_cap * 4);
    }
    cid[0] = (int32_t*)w; w += al((size_t)a->n * 4);
    cid[1] = (int32_t*)w; w += al((size_t)b->n * 4);
    items[0] = (int32_t*)w; w += al((size_t)a->n * 4);
    items[1] = (int32_t*)w; w += al((size_t)b->n * 4);
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (int32_t*)nullptr, (int32_t*)nullptr, (int)cell_cap);
    void* tmp = w;

    k_bbox_init<<<1, 32, 0, st>>>(bba);
    k_bbox_init<<<1, 32, 0, st>>>(bbb);
    k_bbox<<<tl_blocks(a->n, kThreads), kThreads, 0, st>>>(*a, bba);
    k_bbox<<<tl_blocks(b->n, kThreads), kThreads, 0, st>>>(*b, bbb);
    k_grid<<<1, 1, 0, st>>>(bba, bbb, dpc, dim, cell_cap, g);
    int rc = tl_check_launch("k_grid");
    if (rc) return rc;
    const tl_contact_side* side[2] = {a, b};
    for (int k = 0; k < 2; ++k) {
        TL_TRY_CUDA(cudaMemsetAsync(cnt[k], 0, (size_t)cell_cap * 4, st));
        TL_TRY_CUDA(cudaMemsetAsync(cur[k], 0, (size_t)cell_cap * 4, st));
        k_cell_count<<<tl_blocks(side[k]->n, kThreads), kThreads, 0, st>>>(*side[k], g, dim, cnt[k],
                                                                          cid[k]);
        if (cub::DeviceScan::ExclusiveSum(tmp, scan, cnt[k], start[k], (int)cell_cap, st) != cudaSuccess) {
            tl_set_error("contact cell scan failed");
            return TL_ERR_CUDA;
        }
        k_cell_fill<<<tl_blocks(side[k]->n, kThreads), kThreads, 0, st>>>(*side[k], cid[k], start[k],
                                                                         cur[k], items[k]);
    }
    const PairParams p{dpc, k_n, c_n, kfric};
    k_contact_gather<true><<<tl_blocks(a->n, kThreads), kThreads, 0, st>>>(
        *a, *b, g, dim, start[1], cnt[1], items[1], p, acc_a, counters, counters + 1);
    k_contact_gather<false><<<tl_blocks(b->n, kThreads), kThreads, 0, st>>>(
        *b, *a, g, dim, start[0], cnt[0], items[0], p, acc_b, counters, counters + 1);
    return tl_check_launch("k_contact_gather");
}
