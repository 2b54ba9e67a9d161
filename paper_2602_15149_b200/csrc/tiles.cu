// tiles.cu -- spatial reordering and neighbour tiles for the step kernels.
//
// The reference keeps particles in generation order (x-major lattices,
// caseio.py:82-104).  For the fused step kernels the device keeps its own
// order instead: particles sorted along a Morton curve of their
// neighbour-search cells, so that T consecutive particles (one CTA) form a
// compact brick.  Each brick's neighbours are then its own members plus a
// thin halo, which the step kernels stage once into shared memory; every
// pair term then reads shared memory instead of gathering through L1/L2.
//
// Sums stay in the reference's order: each row keeps its neighbours in
// ascending ORIGINAL index (kernel_geom.py:96 lexsort), only renamed to the
// new positions, so results are independent of the reordering.
//
// Built once per body (total Lagrangian: the stencil never changes).
#include <cub/cub.cuh>

#include "tl_common.cuh"

namespace {

constexpr int kThreads = 256;

// spread the low 21 bits of x to every third bit
__device__ __forceinline__ uint64_t spread3(uint64_t x) {
    x &= 0x1fffffull;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

__global__ void k_morton(int64_t n, const double* __restrict__ X, double lo0, double lo1,
                         double lo2, double inv_cell, uint64_t* keys, int32_t* idx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t cx = (uint64_t)max(0.0, floor((X[3 * i] - lo0) * inv_cell));
    const uint64_t cy = (uint64_t)max(0.0, floor((X[3 * i + 1] - lo1) * inv_cell));
    const uint64_t cz = (uint64_t)max(0.0, floor((X[3 * i + 2] - lo2) * inv_cell));
    keys[i] = spread3(cx) << 2 | spread3(cy) << 1 | spread3(cz);
    idx[i] = (int32_t)i;
}

__global__ void k_invert(int64_t n, const int32_t* __restrict__ perm, int32_t* __restrict__ iperm) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < n) iperm[perm[p]] = (int32_t)p;
}

__global__ void k_perm_counts(int64_t n, const int32_t* __restrict__ perm,
                              const int64_t* __restrict__ indptr, int64_t* __restrict__ counts) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < n) {
        const int64_t i = perm[p];
        counts[p] = indptr[i + 1] - indptr[i];
    }
}

__global__ void k_perm_rows(int64_t n, const int32_t* __restrict__ perm,
                            const int32_t* __restrict__ iperm, const int64_t* __restrict__ indptr,
                            const int32_t* __restrict__ indices,
                            const int64_t* __restrict__ indptr_new, int32_t* __restrict__ out) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t i = perm[p];
    const int64_t b = indptr[i], e = indptr[i + 1], o = indptr_new[p];
    for (int64_t k = b; k < e; ++k) out[o + k - b] = iperm[indices[k]];
}

// halo keys: (tile << 32 | neighbour) for neighbours outside the row's tile,
// UINT64_MAX otherwise (sorts last and is dropped)
__global__ void k_halo_keys(int64_t n, int T, const int64_t* __restrict__ indptr,
                            const int32_t* __restrict__ indices, uint64_t* __restrict__ keys) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t tile = p / T;
    // the last tile may be partial: positions >= n are the multi-GPU halo
    // block, never tile members
    const int64_t t0 = tile * T, t1 = min(t0 + T, n);
    for (int64_t k = indptr[p]; k < indptr[p + 1]; ++k) {
        const int64_t q = indices[k];
        keys[k] = (q >= t0 && q < t1) ? ~0ull : ((uint64_t)tile << 32 | (uint64_t)q);
    }
}

// after sort: flag the first occurrence of every (tile, q) key
__global__ void k_halo_flags(int64_t m, const uint64_t* __restrict__ keys, int32_t* __restrict__ flag) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    flag[k] = (keys[k] != ~0ull && (k == 0 || keys[k] != keys[k - 1])) ? 1 : 0;
}

__global__ void k_halo_scatter(int64_t m, const uint64_t* __restrict__ keys,
                               const int32_t* __restrict__ flag, const int64_t* __restrict__ pos,
                               int32_t* __restrict__ halo, int64_t* __restrict__ tile_count) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m || !flag[k]) return;
    halo[pos[k]] = (int32_t)(keys[k] & 0xffffffffull);
    atomicAdd((unsigned long long*)&tile_count[keys[k] >> 32], 1ull);
}

// Lattice offset class of a pair (bond): the reference separation r0 =
// X_i - X_j as an integer multiple q of the body's spacing dp, encoded as
// key = ((qx+R)(2R+1) + qy+R)(2R+1) + qz+R.  TL_KEY_SELF marks the padding
// entries (j == i), TL_KEY_OFF a pair off the lattice (|r0 - q dp| > 1e-6 dp
// or |q| > R): such a body keeps the position path.
#define TL_KEY_SELF 0xffff
#define TL_KEY_OFF 0xfffe
constexpr int kKeyR = 7;

__device__ __forceinline__ uint16_t lattice_key(const double* __restrict__ X, int64_t n_all,
                                                int64_t p, int64_t q, double dp, double inv_dp) {
    int k = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double d = X[a * n_all + p] - X[a * n_all + q];
        const double c = rint(d * inv_dp);
        if (fabs(d - c * dp) > 1e-6 * dp || fabs(c) > kKeyR) return TL_KEY_OFF;
        k = k * (2 * kKeyR + 1) + (int)c + kKeyR;
    }
    return (uint16_t)k;
}

// local slot of every pair, in the group-interleaved sliced layout:
// slot(w, k, lane) at soff[w] + (k/G)*32*G + lane*G + k%G; padding = own slot.
// keys (optional): the pair's lattice offset class key in the same layout.
__global__ void k_slots(int64_t n, int T, int G, int shift, const int64_t* __restrict__ indptr,
                        const int32_t* __restrict__ indices, const int64_t* __restrict__ hoff,
                        const int32_t* __restrict__ halo, const uint16_t* __restrict__ hslot,
                        const int64_t* __restrict__ soff, uint16_t* __restrict__ slots,
                        const double* __restrict__ X, int64_t n_all, double dp,
                        uint16_t* __restrict__ keys) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nw = (n + 31) / 32;
    const int64_t w = p >> 5;
    if (w >= nw) return;
    const int lane = (int)(p & 31);
    const int64_t tile = p / T;
    const int64_t t0 = tile * T;
    const int64_t base = soff[w];
    const int64_t len = (soff[w + 1] - base) / 32;
    const int64_t rb = p < n ? indptr[p] : 0;
    const int64_t rl = p < n ? indptr[p + 1] - rb : 0;
    const uint16_t self = (uint16_t)(p - t0);
    const int32_t* hs = halo + (p < n ? hoff[tile] : 0);
    const uint16_t* hsl = hslot + (p < n ? hoff[tile] : 0);
    const int64_t hn = p < n ? hoff[tile + 1] - hoff[tile] : 0;
    const double inv_dp = keys ? 1.0 / dp : 0.0;
    for (int64_t k = 0; k < len; ++k) {
        uint16_t s = self;
        uint16_t key = TL_KEY_SELF;
        if (k < rl) {
            const int64_t q = indices[rb + k];
            if (q >= t0 && q < t0 + T && q < n) {
                s = (uint16_t)(q - t0);
            } else {
                int64_t lo = 0, hi = hn;
                while (lo < hi) {
                    const int64_t m = (lo + hi) >> 1;
                    if (hs[m] < q) lo = m + 1; else hi = m;
                }
                s = hsl[lo];
            }
            if (keys) key = lattice_key(X, n_all, p, q, dp, inv_dp);
        }
        const int64_t e = base + (k / G) * 32 * G + lane * G + (k % G);
        slots[e] = (uint16_t)(s << shift);
        if (keys) keys[e] = key;
    }
}

// bond-class slot entries: (class << 10) | slot, from the plain slots
// (slot << shift) and the per-key class table
__global__ void k_class_slots(int64_t m, int shift, const uint16_t* __restrict__ keys,
                              const int16_t* __restrict__ cls_of_key, uint16_t* __restrict__ slots) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= m) return;
    const uint16_t key = keys[e];
    const int c = key == TL_KEY_SELF ? 0 : cls_of_key[key];
    slots[e] = (uint16_t)((c << 10) | (slots[e] >> shift));
}

// Shared-memory slot of every halo entry of every tile.  A quarter-warp's
// 128-bit shared loads hit distinct bank groups when the 8 slots it reads
// are distinct mod 8.  Members sit at slot p - t0 (== p mod 8, tiles are
// multiples of 8); giving halo particle q a slot == q (mod 8) as well,
// T + 8*rank + (q & 7) with rank = its order within that residue class,
// keeps a Morton-ordered warp's k-th neighbours (a translated 2x2x2 brick
// per quarter-warp) conflict-free off the tile too.  A tile whose aligned
// extent would exceed `cap` (> 0) is packed densely instead, so a few
// fragmented tiles do not set the shared-memory size of every CTA; res = 1
// packs every tile densely.  One thread per tile; extent[t] = slots used - T.
__global__ void k_hslots(int64_t ntile, int T, int res, int cap, const int64_t* __restrict__ hoff,
                         const int32_t* __restrict__ halo, uint16_t* __restrict__ hslot,
                         int32_t* __restrict__ extent) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= ntile) return;
    const int64_t k0 = hoff[t], k1 = hoff[t + 1];
    bool aligned = res == 8;
    if (aligned && cap > 0) {
        int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t k = k0; k < k1; ++k) {
            const int r = halo[k] & 7;
#pragma unroll
            for (int q = 0; q < 8; ++q) cnt[q] += (q == r);
        }
        int top = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (cnt[q]) top = max(top, 8 * (cnt[q] - 1) + q + 1);
        aligned = top <= cap;
    }
    int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int top = 0;
    for (int64_t k = k0; k < k1; ++k) {
        int slot;
        if (aligned) {
            const int r = halo[k] & 7;
            int c = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q == r) c = cnt[q]++;
            slot = 8 * c + r;
        } else {
            slot = (int)(k - k0);
        }
        hslot[k] = (uint16_t)(T + slot);
        top = max(top, slot + 1);
    }
    extent[t] = top;
}

// Staged position record of every slot of every tile, built once: the
// reference positions relative to the tile's first member (FP32; absolute in
// FP64) and the particle's mass-like weight (w), in slot order, so the step
// kernels copy a contiguous block instead of gathering FP64 planes.
// toff[t] = first record of tile t; holes stay zero.
template <typename R>
__global__ void k_tile_pos(int64_t n, int64_t n_all, int T, int64_t ntile,
                           const int64_t* __restrict__ hoff, const int32_t* __restrict__ halo,
                           const uint16_t* __restrict__ hslot, const int64_t* __restrict__ toff,
                           const double* __restrict__ X, const double* __restrict__ w, int rel,
                           R* __restrict__ out) {
    const int64_t t = blockIdx.x;
    if (t >= ntile) return;
    const int64_t p0 = t * T;
    const double ox = rel ? X[p0] : 0.0, oy = rel ? X[n_all + p0] : 0.0,
                 oz = rel ? X[2 * n_all + p0] : 0.0;
    const int64_t k0 = hoff[t], H = hoff[t + 1] - k0;
    R* o = out + 4 * toff[t];
    for (int64_t s = threadIdx.x; s < T + H; s += blockDim.x) {
        int64_t q;
        int64_t d;
        if (s < T) {
            if (p0 + s >= n) continue;
            q = p0 + s;
            d = s;
        } else {
            q = halo[k0 + s - T];
            d = hslot[k0 + s - T];
        }
        o[4 * d] = R(X[q] - ox);
        o[4 * d + 1] = R(X[n_all + q] - oy);
        o[4 * d + 2] = R(X[2 * n_all + q] - oz);
        o[4 * d + 3] = w ? R(w[q]) : R(0);
    }
}

}  // namespace

extern "C" int tl_reorder(tl_stream_t st_, int64_t n, const double* X, const double* lo,
                          double cell, int32_t* perm, int32_t* iperm) {
    cudaStream_t st = (cudaStream_t)st_;
    if (n <= 0) return TL_OK;
    uint64_t *kin, *kout;
    int32_t* idx;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (int32_t*)nullptr, (int32_t*)nullptr, n, 0, 63, st);
    char* pool;
    const size_t a = ((size_t)n * 8 + 255) & ~size_t(255);
    const size_t b = ((size_t)n * 4 + 255) & ~size_t(255);
    TL_TRY_CUDA(cudaMallocAsync((void**)&pool, 2 * a + b + tmp_bytes, st));
    kin = (uint64_t*)pool;
    kout = (uint64_t*)(pool + a);
    idx = (int32_t*)(pool + 2 * a);
    void* tmp = pool + 2 * a + b;
    k_morton<<<tl_blocks(n, kThreads), kThreads, 0, st>>>(n, X, lo[0], lo[1], lo[2], 1.0 / cell,
                                                          kin, idx);
    int rc = tl_check_launch("k_morton");
    if (!rc) {
        cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, idx, perm, n, 0, 63, st);
        if (e != cudaSuccess) {
            tl_set_error("morton sort: %s", cudaGetErrorString(e));
            rc = TL_ERR_CUDA;
        }
    }
    if (!rc) {
        k_invert<<<tl_blocks(n, kThreads), kThreads, 0, st>>>(n, perm, iperm);
        rc = tl_check_launch("k_invert");
    }
    cudaFreeAsync(pool, st);
    return rc;
}

extern "C" int tl_csr_permute_counts(tl_stream_t st, int64_t n, const int32_t* perm,
                                     const int64_t* indptr, int64_t* counts) {
    if (n <= 0) return TL_OK;
    k_perm_counts<<<tl_blocks(n, kThreads), kThreads, 0, (cudaStream_t)st>>>(n, perm, indptr, counts);
    return tl_check_launch("k_perm_counts");
}

extern "C" int tl_csr_permute(tl_stream_t st, int64_t n, const int32_t* perm, const int32_t* iperm,
                              const int64_t* indptr, const int32_t* indices,
                              const int64_t* indptr_new, int32_t* indices_new) {
    if (n <= 0) return TL_OK;
    k_perm_rows<<<tl_blocks(n, kThreads), kThreads, 0, (cudaStream_t)st>>>(
        n, perm, iperm, indptr, indices, indptr_new, indices_new);
    return tl_check_launch("k_perm_rows");
}

extern "C" int tl_tile_halo(tl_stream_t st_, int64_t n, int32_t T, const int64_t* indptr,
                            const int32_t* indices, int64_t nnz, int32_t* halo,
                            int64_t* tile_count, int64_t* n_halo) {
    cudaStream_t st = (cudaStream_t)st_;
    if (n <= 0 || nnz <= 0) return TL_OK;
    const int64_t ntile = (n + T - 1) / T;
    size_t sort_bytes = 0, scan_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, nnz,
                                   0, 64, st);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int32_t*)nullptr, (int64_t*)nullptr, nnz, st);
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    const size_t kb = al((size_t)nnz * 8), fb = al((size_t)nnz * 4), pb = al((size_t)nnz * 8);
    char* pool;
    TL_TRY_CUDA(cudaMallocAsync((void**)&pool, 2 * kb + fb + pb + al(sort_bytes) + al(scan_bytes) + 256, st));
    uint64_t* k0 = (uint64_t*)pool;
    uint64_t* k1 = (uint64_t*)(pool + kb);
    int32_t* flag = (int32_t*)(pool + 2 * kb);
    int64_t* pos = (int64_t*)(pool + 2 * kb + fb);
    void* stmp = pool + 2 * kb + fb + pb;
    void* ctmp = (char*)stmp + al(sort_bytes);
    int rc = TL_OK;
    k_halo_keys<<<tl_blocks(n, kThreads), kThreads, 0, st>>>(n, T, indptr, indices, k0);
    rc = tl_check_launch("k_halo_keys");
    if (!rc && cub::DeviceRadixSort::SortKeys(stmp, sort_bytes, k0, k1, nnz, 0, 64, st) != cudaSuccess) {
        tl_set_error("halo sort failed");
        rc = TL_ERR_CUDA;
    }
    if (!rc) {
        k_halo_flags<<<tl_blocks(nnz, kThreads), kThreads, 0, st>>>(nnz, k1, flag);
        rc = tl_check_launch("k_halo_flags");
    }
    if (!rc && cub::DeviceScan::ExclusiveSum(ctmp, scan_bytes, flag, pos, nnz, st) != cudaSuccess) {
        tl_set_error("halo scan failed");
        rc = TL_ERR_CUDA;
    }
    if (!rc) {
        cudaMemsetAsync(tile_count, 0, sizeof(int64_t) * ntile, st);
        if (halo) {
            k_halo_scatter<<<tl_blocks(nnz, kThreads), kThreads, 0, st>>>(nnz, k1, flag, pos, halo,
                                                                         tile_count);
            rc = tl_check_launch("k_halo_scatter");
        }
    }
    if (!rc && n_halo) {
        // total = pos[last] + flag[last]
        int64_t last_pos = 0;
        int32_t last_flag = 0;
        cudaMemcpyAsync(&last_pos, pos + nnz - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&last_flag, flag + nnz - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        *n_halo = last_pos + last_flag;
    }
    cudaFreeAsync(pool, st);
    return rc;
}

extern "C" int tl_tile_hslots(tl_stream_t st, int64_t ntile, int32_t T, int32_t res, int32_t cap,
                              const int64_t* hoff, const int32_t* halo, uint16_t* hslot,
                              int32_t* extent) {
    if (ntile <= 0) return TL_OK;
    if (res != 1 && res != 8) {
        tl_set_error("tl_tile_hslots: res must be 1 or 8");
        return TL_ERR_ARG;
    }
    if (T % 8) {
        tl_set_error("tl_tile_hslots: tile size must be a multiple of 8");
        return TL_ERR_ARG;
    }
    k_hslots<<<tl_blocks(ntile, 128), 128, 0, (cudaStream_t)st>>>(ntile, T, res, cap, hoff, halo,
                                                                 hslot, extent);
    return tl_check_launch("k_hslots");
}

extern "C" int tl_tile_pos(tl_stream_t st, int64_t n, int64_t n_all, int32_t T, int64_t ntile,
                           const int64_t* hoff, const int32_t* halo, const uint16_t* hslot,
                           const int64_t* toff, const double* X, const double* w, int32_t precision,
                           void* out) {
    if (ntile <= 0) return TL_OK;
    cudaStream_t s = (cudaStream_t)st;
    if (precision == 4)
        k_tile_pos<float><<<(unsigned)ntile, 256, 0, s>>>(n, n_all, T, ntile, hoff, halo, hslot, toff,
                                                          X, w, 1, (float*)out);
    else
        k_tile_pos<double><<<(unsigned)ntile, 256, 0, s>>>(n, n_all, T, ntile, hoff, halo, hslot, toff,
                                                           X, w, 0, (double*)out);
    return tl_check_launch("k_tile_pos");
}

extern "C" int tl_tile_slots(tl_stream_t st, int64_t n, int32_t T, int32_t G, int32_t shift,
                             const int64_t* indptr, const int32_t* indices, const int64_t* hoff,
                             const int32_t* halo, const uint16_t* hslot, const int64_t* soff,
                             uint16_t* slots) {
    return tl_tile_slots_keyed(st, n, T, G, shift, indptr, indices, hoff, halo, hslot, soff, slots,
                               nullptr, 0, 0.0, nullptr);
}

extern "C" int tl_tile_slots_keyed(tl_stream_t st, int64_t n, int32_t T, int32_t G, int32_t shift,
                                   const int64_t* indptr, const int32_t* indices,
                                   const int64_t* hoff, const int32_t* halo, const uint16_t* hslot,
                                   const int64_t* soff, uint16_t* slots, const double* X,
                                   int64_t n_all, double dp, uint16_t* keys) {
    if (n <= 0) return TL_OK;
    if (shift < 0 || shift > 8) {
        tl_set_error("tl_tile_slots: shift out of range");
        return TL_ERR_ARG;
    }
    if (keys && (!X || !(dp > 0.0))) {
        tl_set_error("tl_tile_slots_keyed: keys need positions and dp > 0");
        return TL_ERR_ARG;
    }
    const int64_t nt = ((n + 31) / 32) * 32;
    k_slots<<<tl_blocks(nt, kThreads), kThreads, 0, (cudaStream_t)st>>>(
        n, T, G, shift, indptr, indices, hoff, halo, hslot, soff, slots, X, n_all, dp, keys);
    return tl_check_launch("k_slots");
}

extern "C" int tl_class_slots(tl_stream_t st, int64_t m, int32_t shift, const uint16_t* keys,
                              const int16_t* cls_of_key, uint16_t* slots) {
    if (m <= 0) return TL_OK;
    k_class_slots<<<tl_blocks(m, kThreads), kThreads, 0, (cudaStream_t)st>>>(m, shift, keys,
                                                                          cls_of_key, slots);
    return tl_check_launch("k_class_slots");
}
