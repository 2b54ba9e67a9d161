/*
 * tlsph.h -- C ABI of libtlsph.so, the B200 (sm_100a) TLSPH hot path.
 *
 * Plain C: device pointers, sizes and scalars only; no torch or C++ types.
 * Every function is asynchronous on the given CUDA stream and returns 0 or a
 * negative TL_ERR_* code; tl_last_error() gives the message (per host
 * thread).  Numeric events the reference reports as return values (degenerate
 * counts, first non-SPD particle, non-convergence) are accumulated into
 * caller-provided DEVICE words and read at sync points, so no call blocks.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/solidsph/<file>:<line>).  INTEGRATION.md shows the
 * ctypes binding a solidsph maintainer would add.
 */
#ifndef TLSPH_H
#define TLSPH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* tl_stream_t; /* a cudaStream_t; NULL = legacy default stream */

enum {
    TL_OK = 0,
    TL_ERR_ARG = -1,
    TL_ERR_CUDA = -2,
    TL_ERR_UNSUPPORTED = -3,
    TL_ERR_CASE = -4
};

#define TL_ABI_VERSION 11

int tl_abi_version(void);
/* sizeof of the ABI structs, for binding checks: 0 tl_body, 1 tl_clock,
 * 2 tl_bc, 3 tl_prog, 4 tl_notch, 5 tl_nb_params, 6 tl_dtinfo */
int64_t tl_struct_size(int which);
const char* tl_last_error(void);
int tl_device_sync(void);

/* ---------------------------------------------------------------------------
 * Backend-plugin kernels (reference backends/reference.py:18-244 and
 * backends/fast.py:111-469).  Same argument meaning as the reference plugin:
 * FP64, row-major (n,3) vectors and (n,3,3) tensors, int64 CSR.  Outputs are
 * caller-allocated and written in place.  One CUDA thread per particle sums
 * its neighbours sequentially in CSR order, like the reference.
 * ------------------------------------------------------------------------- */

/* F_i = I + sum_j V0_j (u_j-u_i) (x) grad0_ij; identity when gated and
 * s_i <= s_l.  Replaces backends.deformation_gradient (reference.py:18). */
int tl_deformation_gradient(tl_stream_t st, int64_t n, const int64_t* indptr,
                            const int64_t* indices, const double* grad0, const double* u,
                            const double* V0, const double* s, double s_l, int gated,
                            double* out);

/* Brookshaw Laplacian.  Replaces backends.sph_laplacian (reference.py:32). */
int tl_sph_laplacian(tl_stream_t st, int64_t n, const int64_t* indptr, const int64_t* indices,
                     const double* grad0, const double* r0, const double* r0norm,
                     const double* V0, const double* f, double* out);

/* Corrected gradient.  Replaces backends.sph_gradient (reference.py:42). */
int tl_sph_gradient(tl_stream_t st, int64_t n, const int64_t* indptr, const int64_t* indices,
                    const double* grad0, const double* V0, const double* f, double* out);

/* Momentum with artificial viscosity; *n_bad (device) += degenerate count.
 * Replaces backends.momentum (reference.py:52). */
int tl_momentum(tl_stream_t st, int64_t n, const int64_t* indptr, const int64_t* indices,
                const double* grad0, const double* grad0r, const double* r0,
                const double* r0norm, const double* P, const double* m0, double rho0,
                const double* v, double h, double c0, double beta1, double beta2,
                const double* F, double* out, int64_t* n_bad);

/* SVK (+ spectral split when fracture); *n_noconv (device) += count.
 * Replaces backends.svk_batch (reference.py:94). */
int tl_svk_batch(tl_stream_t st, int64_t n, const double* F, double lam, double mu,
                 const double* s, int fracture, double* out_S, double* out_psi,
                 double* out_psip, int64_t* n_noconv);

/* Neo-Hookean; *n_bad (device) += degenerate count.
 * Replaces backends.nh_batch (reference.py:119). */
int tl_nh_batch(tl_stream_t st, int64_t n, const double* F, double kappa, double mu,
                const double* s, int fracture, double* out_S, double* out_psi,
                double* out_psip, int64_t* n_bad);

/* J2 radial return, Cp and epbar updated in place.  counters (device):
 * [0] += degenerate count, [1] = min(first non-SPD index) (init to INT64_MAX).
 * As in the reference, a non-SPD update leaves the state uncommitted.
 * Replaces backends.j2_batch (reference.py:151). */
int tl_j2_batch(tl_stream_t st, int64_t n, const double* F, double* Cp, double* epbar,
                double mu, double kappa, double sigma_y0, double H_hard, double* out_S,
                double* out_psi, double* out_dwp, int64_t* counters, uint8_t* scratch);

/* Penalty contact over candidate pairs, accumulated in pair order like the
 * reference; *n_warn (device) += coincident count.  scratch: 3*npairs doubles.
 * Replaces backends.contact_pair_accumulate (reference.py:211). */
int tl_contact_pair_accumulate(tl_stream_t st, const double* xa, const double* va,
                               const double* ma, const double* xb, const double* vb,
                               const double* mb, int64_t npairs, const int64_t* pairs,
                               double dp_contact, double k_n, double c_n, double kfric,
                               double* out_aa, double* out_ab, int64_t* n_warn,
                               double* scratch);

/* Batched symmetric 3x3 Jacobi (descending), sweeps per matrix.
 * Replaces fast._eig3_jacobi (fast.py:45). */
int tl_eig3_jacobi(tl_stream_t st, int64_t n, const double* A, double* w, double* Q,
                   int32_t* sweeps);

/* ---------------------------------------------------------------------------
 * Reference-configuration neighbour build (kernel_geom.py:65-261).
 * Cell list radix-sorted by x-major cell key, exact inclusion tests in the
 * reference's FP64 operation order, notch severing on directed pairs, CSR
 * rows in ascending partner index.
 * ------------------------------------------------------------------------- */
typedef struct {
    double origin[3], nhat[3], e1[3], e2[3];
    double poly[4][2];
    double tol_plane, tol_poly;
} tl_notch;

typedef struct {
    int64_t n;
    const double* X;      /* (n,3) reference positions, device */
    int mode;             /* 0 = radial |d|^2 < (2h)^2, 1 = nbsrange window */
    double h;             /* smoothing length */
    double win;           /* nbsrange window (mode 1) */
    double lo[3];         /* bounding-box minimum */
    double cell;          /* cell edge (>= cutoff) */
    int64_t dims[3];      /* cells per axis */
    int n_notch;
    const tl_notch* notches; /* host array of n_notch frames */
} tl_nb_params;

typedef struct tl_nb_plan tl_nb_plan;

/* sort particles into cells.  Replaces the cKDTree prefilter (kernel_geom.py:76-86). */
int tl_nb_plan_create(tl_stream_t st, const tl_nb_params* p, tl_nb_plan** out);
/* counts[i] = kept partners of i after notch severing (device int64[n]). */
int tl_nb_count(tl_nb_plan* plan, int64_t* counts);
/* CSR fill with ascending partners; indptr (device int64[n+1]) from counts.
 * Replaces build_pairs + sever_notch_bonds + _csr_from_pairs
 * (kernel_geom.py:65-173). */
int tl_nb_fill(tl_nb_plan* plan, const int64_t* indptr, int32_t* indices);
int tl_nb_plan_destroy(tl_nb_plan* plan);

/* First-order correction L_i = A_i^-1 with the cond_2 >= 1e8 identity
 * fallback; *fallbacks (device) += count.  L: (n,3,3) FP64.
 * Replaces correction_matrices (kernel_geom.py:176-205). */
int tl_correction(tl_stream_t st, int64_t n, const int64_t* indptr, const int32_t* indices,
                  const double* X, const double* V0, double h, double alpha, int kind, int dim,
                  int correction, double* L, int64_t* fallbacks);

/* Per-pair arrays of the reference Adjacency (kernel_geom.py:228-261):
 * rows, r0 = Xi-Xj, r0norm, w0, grad0 = L_i gb, grad0r = -L_j gb (== grad0
 * of the reverse pair).  Any output may be NULL. */
int tl_adjacency_expand(tl_stream_t st, int64_t n, const int64_t* indptr,
                        const int32_t* indices, const double* X, const double* L, double h,
                        double alpha, int kind, int64_t* rows, double* r0, double* r0norm,
                        double* w0, double* grad0, double* grad0r);

/* Sliced-ELL (32 particles per slice, lane-interleaved) copy of the CSR for
 * coalesced neighbour-index loads in the fused step kernels.
 * tl_sell_lengths: slen[w] = max row length in slice w rounded up to a
 * multiple of TL_SELL_GROUP (device int32[nw]).
 * tl_sell_fill: soff (device int64[nw+1], exclusive scan of 32*slen), sidx
 * (device int32[soff[nw]]); padding slots hold the row's own index, whose
 * pair terms vanish exactly (r0 = 0). */
#define TL_SELL_GROUP 4
int tl_sell_lengths(tl_stream_t st, int64_t n, const int64_t* indptr, int32_t* slen);
int tl_sell_fill(tl_stream_t st, int64_t n, const int64_t* indptr, const int32_t* indices,
                 const int64_t* soff, int32_t* sidx);

/* ---------------------------------------------------------------------------
 * Device particle order and neighbour tiles (tiles.cu).  The step kernels
 * run on particles sorted along a Morton curve of their cells so a CTA's
 * neighbours are its own members plus a thin halo staged in shared memory.
 * Rows keep ascending ORIGINAL partner order: sums match the reference's.
 * ------------------------------------------------------------------------- */
/* perm[p] = original index at device position p, iperm its inverse */
int tl_reorder(tl_stream_t st, int64_t n, const double* X, const double* lo, double cell,
               int32_t* perm, int32_t* iperm);
int tl_csr_permute_counts(tl_stream_t st, int64_t n, const int32_t* perm, const int64_t* indptr,
                          int64_t* counts);
int tl_csr_permute(tl_stream_t st, int64_t n, const int32_t* perm, const int32_t* iperm,
                   const int64_t* indptr, const int32_t* indices, const int64_t* indptr_new,
                   int32_t* indices_new);
/* halo of every tile of T particles (capacity nnz); tile_count[ntile];
 * *n_halo = total (host) */
int tl_tile_halo(tl_stream_t st, int64_t n, int32_t T, const int64_t* indptr,
                 const int32_t* indices, int64_t nnz, int32_t* halo, int64_t* tile_count,
                 int64_t* n_halo);
/* shared-memory slot of every halo entry: res = 8 puts halo particle q at a
 * slot == q (mod 8), the residue of a member's slot, so a quarter-warp's
 * 128-bit loads of translated neighbours avoid bank conflicts (tiles whose
 * aligned extent exceeds cap > 0 are packed densely); res = 1 packs every
 * tile densely.  extent[t] (device int32[ntile]) = halo slots tile t uses */
int tl_tile_hslots(tl_stream_t st, int64_t ntile, int32_t T, int32_t res, int32_t cap,
                   const int64_t* hoff, const int32_t* halo, uint16_t* hslot, int32_t* extent);
/* staged position records (x, y, z, w) of every slot of every tile, in slot
 * order from toff[t] (device int64[ntile+1]); FP32 (precision 4): relative to
 * the tile's first member, FP64: absolute; w = per-particle weight or 0 when
 * w == NULL.  out: device Real[4*toff[ntile]], zeroed by the caller */
int tl_tile_pos(tl_stream_t st, int64_t n, int64_t n_all, int32_t T, int64_t ntile,
                const int64_t* hoff, const int32_t* halo, const uint16_t* hslot, const int64_t* toff,
                const double* X, const double* w, int32_t precision, void* out);
/* per-pair shared-memory slots of the tiled step kernels, stored as
 * slot << shift (shift 4: the byte offset of the slot's FP32 position
 * record; FP64 records are two such units) */
int tl_tile_slots(tl_stream_t st, int64_t n, int32_t T, int32_t G, int32_t shift,
                  const int64_t* indptr, const int32_t* indices, const int64_t* hoff,
                  const int32_t* halo, const uint16_t* hslot, const int64_t* soff, uint16_t* slots);
/* the same, plus keys (same layout): every pair's lattice offset class key,
 * ((qx+7)*15 + qy+7)*15 + qz+7 for r0 = X_i - X_j = q dp (device FP64 planes X
 * of stride n_all); 0xffff = self padding, 0xfffe = off the lattice.  The
 * reference configuration is fixed (kernel_geom.py:1-6), so r0 of every pair
 * is too: a lattice body's pairs take a handful of separations. */
int tl_tile_slots_keyed(tl_stream_t st, int64_t n, int32_t T, int32_t G, int32_t shift,
                        const int64_t* indptr, const int32_t* indices, const int64_t* hoff,
                        const int32_t* halo, const uint16_t* hslot, const int64_t* soff,
                        uint16_t* slots, const double* X, int64_t n_all, double dp,
                        uint16_t* keys);
/* rewrite m slot entries (slot << shift) as (cls_of_key[key] << 10) | slot
 * (class 0 for the self padding) */
int tl_class_slots(tl_stream_t st, int64_t m, int32_t shift, const uint16_t* keys,
                   const int16_t* cls_of_key, uint16_t* slots);

/* ---------------------------------------------------------------------------
 * Fused device-resident step (stepper.py:77-209, dynamics.py:28-217,
 * constitutive.py:168-199, fracture.py:12-83).
 * ------------------------------------------------------------------------- */

#define TL_MAX_BC 32
#define TL_MAX_PROG 64

/* expression program table (bytecode from expr.compile_program) */
typedef struct {
    const int32_t* code;   /* (len,2) opcode/operand pairs, device */
    const double* consts;  /* device */
    int32_t len;
    int32_t pad;
} tl_prog;

typedef struct {
    int32_t kind;          /* 0 = velocity, 1 = force */
    int32_t ftype;         /* force type 1|2|3 */
    int32_t bit;           /* membership bit in bcmask, -1 = whole body */
    int32_t has_const[3];
    int32_t prog[3];       /* program index or -1 (axis untouched unless const) */
    double cval[3];
    double tst, tend;
    /* skip guard of a whole-body entry (expr.skip_guard_after): for t > gt the
     * entry is skip for every particle where `var gop gc` is false (var in
     * x0 y0 z0 x y z ux uy uz, expr.VARIABLES order; gop 0 <, 1 >, 2 <=, 3 >=),
     * so the step evaluates it on the other particles only; gvar -1 = none */
    int32_t gvar, gop;
    double gc, gt;
} tl_bc;

/* device clock: time integration state kept on the device so steps never
 * wait for the host (stepper.py:221-263 semantics) */
typedef struct {
    double t;           /* current time */
    double dt;          /* dt of the step in flight */
    double next_out;    /* next output boundary */
    double t_max;
    double eps;         /* 1e-12*max(t_max,1) */
    double dt_override; /* <0: adaptive */
    double cfl;
    int64_t step;       /* step_index */
    int64_t max_steps;  /* <0: unlimited */
    int32_t halted;     /* 0 run, 1 finished, 2 output due, 3 max_steps, 4 dt collapsed,
                           5 error raised inside the step, 6 non-finite state at a
                           64-step commit (stepper.py:203-209) */
    int32_t out_step;   /* this step ends on an output boundary: mirror F, S, psi, a */
    int32_t err;        /* errors of the step in flight: bit 0 stress (eigen / non-SPD:
                           raised before momentum, constitutive.py:177-194, so pass B
                           skips), bit 1 acceleration / expression / restrictphi; the
                           step is not committed and the clock halts (5) */
    int32_t nf_now;     /* this step left some u or v non-finite */
} tl_clock;

/* Per-body device view.  Layout (Real = float | double per `precision`):
 *   planes  : p[c * n_all + i]   own-particle fields, perfectly coalesced
 *   records : p[R * i + c]       fields gathered from neighbours, one
 *                                128-bit load per 4 values
 * Neighbour indices may reach n_all > n (halo copies on multi-GPU slabs). */
typedef struct {
    int64_t n;              /* particles updated by this call */
    int64_t n_all;          /* owned + halo; plane stride */
    int32_t dim, model, fracture, visc, precision /* 4 | 8 */, kind;
    int32_t uniform, write_out, store_a, nbc, mk, restrict_prog;
    int32_t bc_whole;       /* some BC targets the whole body (during [bcw_lo, bcw_hi]) */
    int32_t unroll;         /* gather group (1 = plain loop, 2, 4); 0 = default */
    /* material / kernel constants (core.py:95-139) */
    double h, inv_h, alpha, rho0, lam, mu, kappa, c0, beta1, beta2;
    double Gc, eps0, s_l, sigma_y0, H_hard, V0c, m0c, dp_body, jac_tol;
    double inv_Gc, inv_eps0, inv_c0;   /* reciprocals (no per-particle divisions) */
    double f0[3];
    /* neighbours: sliced ELL, 32 particles per slice, lane-interleaved;
     * wlen[w] = longest real row of slice w (slices are padded to 4) */
    const int64_t* soff;
    const int32_t* sidx;
    const int32_t* wlen;
    /* shared-memory tiles (tile > 0): CTA = `tile` consecutive particles;
     * hoff[t]..hoff[t+1] indexes its halo particles in `halo`, staged at
     * shared slots `hslot`; slots are uint16 local indices (member
     * p - t*tile, or the halo entry's hslot), grouped TL_SELL_GROUP per lane,
     * same slice offsets as sidx.  hmax = max halo slot extent over tiles;
     * every tile uses the plane stride tile + hmax */
    int32_t tile, hmax;
    int32_t slmax;          /* max slot-table entries of one tile (its warps' slices) */
    int32_t bsplit;         /* tiled FP32 3D pass B: 1, or 4 threads per member, each
                               summing a quarter of the row (high-k stencils) */
    int32_t ncls;           /* bond classes (FP32, uniform lattice bodies): 0 = the pair
                               geometry comes from staged positions; > 0 = slots hold
                               (class << 10) | slot and bcls holds ncls entries */
    int32_t lpp;            /* L2-gather pass B (tile 0 or the untiled pass B): 1, 2, 4 or
                               8 lanes per particle, each summing every lpp-th group of the
                               row (small FP32 bodies: one latency chain per lane is shorter);
                               0 reads as 1 */
    const int64_t* hoff;
    const int32_t* halo;
    const uint16_t* slots;
    const uint16_t* hslot;
    /* tile list (multi-GPU split launches): when non-NULL, a tiled pass runs
     * tiles tlist[tbase .. tbase + tcount) instead of all tiles */
    const int32_t* tlist;
    int64_t tbase, tcount;
    /* staged position records (tl_tile_pos) with V0 (pass A) and m0 (pass B)
     * weights -- the same array when uniform; toff[t] = first record of tile t */
    const int64_t* toff;
    const void* tpos_a;
    const void* tpos_b;
    /* bond-class table, 8 Reals per class: (W, kappa, U, 0) with W = w(r) r0,
     * kappa = 1 / (w(r) (r^2 + 0.001 h^2)) (0 when w = 0), U = r0 / r^2, for the
     * class's reference separation r0 = q dp (q an integer lattice offset;
     * class 0 = the row's self padding, all zero).  The kernel shape w(r) as
     * in the pair loops, the per-body constant applied once per particle. */
    const void* bcls;       /* float (FP32 bodies) or double (FP64) */
    /* geometry */
    const double* Xs;       /* FP64 planes x,y,z */
    const void* L;          /* 9 planes, correction matrix L_i */
    const double* V0;       /* per particle when !uniform */
    const double* m0;
    /* contact acceleration (3 FP64 planes, stride n_all) added before f0, or NULL */
    const double* ac;
    /* state */
    void* us;               /* records of 4: ux uy uz s        (pass-A gather) */
    void* rb;               /* records of 12 (pass-B gather): PL00 PL10 PL01 PL11 | PL02 PL12
                               PL20 PL21 | vx vy vz PL22 (rows 0, 1 interleaved by column) */
    void* v;                /* 3 planes */
    void* al;               /* 9 planes: det(F) F^-1 L_i (viscosity) */
    void* sdot;             /* plane */
    void* sddot;            /* plane */
    void* Hh;               /* plane, history functional */
    void* Cpd;              /* 6 planes, Cp - I: xx yy zz xy xz yz (J2) */
    void* epbar;            /* plane */
    void* a;                /* 3 planes (symplectic predictor / output) */
    /* optional FP64 host-layout outputs when write_out: (n,3,3) / (n,) */
    double* F_out;
    double* S_out;
    double* psi_out;
    double* psip_out;
    const int32_t* perm;    /* device order -> caller's particle index (NULL = identity);
                               error words report caller indices */
    /* boundary conditions */
    const uint32_t* bcmask;
    const tl_bc* bcs;       /* device array of nbc */
    const tl_prog* progs;   /* device program table */
    /* device words */
    tl_clock* clock;
    unsigned long long* red;   /* [0] max|v|^2 bits, [1] max|a|^2 bits */
    int64_t* counters;         /* [0] degenerate, [1] eig noconv, [2] first non-SPD,
                                  [3] first non-finite accel, [4] expr error code,
                                  [5] restrictphi out of [0,1], [6] step of [3],
                                  [7] first step with non-finite u or v */
    double* pw_partial;        /* plastic-work block partials (J2) */
    /* lattice-brick mode (3D lattice bodies with wide stencils; brick[0] = 0:
     * off).  The CTA of brick t owns the lattice cells [o, o + brick) and
     * stages the gather records of the (brick + 2 reach) box of cells around
     * them, addressed by cell: no neighbour or slot tables.  Particle i's
     * bonds are the set bits of bmask (class c = bit c, classes in the
     * reference's CSR summation order); class c's partner sits at i's box
     * cell + bdelta[c], and bbcls holds its geometry as the bond-class table
     * above.  Grid = nbrick[0] * nbrick[1] * nbrick[2] CTAs of brick[0] *
     * brick[1] * brick[2] threads, brick index z fastest. */
    int32_t brick[3];          /* cells per brick and axis */
    int32_t nbrick[3];         /* bricks per axis */
    int32_t cells[3];          /* lattice cells per axis of the body's box */
    int32_t reach;             /* max |q| per axis over the classes */
    int32_t nbcls;             /* bond classes of the brick table */
    int32_t nmask;             /* bond-mask words per particle */
    const int32_t* cellmap;    /* cell (x slowest, z fastest) -> device position, -1 empty */
    const uint32_t* bmask;     /* nmask planes of n_all words */
    const int32_t* bdelta;     /* per class: box-cell offset of the partner */
    const void* bbcls;         /* per class 2 Real4: (W, kappa), (U, 0) */
    /* HOST copies of bdelta / bbcls: the launch passes the class table to the
     * brick kernels as a kernel parameter (constant bank: the loop index is
     * warp-uniform, so every class load is a broadcast); at most
     * TL_BRICK_MAX_CLASSES classes */
    const int32_t* bdelta_host;
    const void* bbcls_host;
    /* register blocking of the brick kernels: cpt cells per thread along z
     * (1 or 2); boxz = the staged box's z extent (brick[2] + 2 reach, padded
     * odd for cpt = 2: conflict-free records); with cpt = 2, ncol columns of
     * the stencil (HOST array of 4 ints each: box offset of the (qx, qy)
     * column, qz_lo, qz_hi, class of qz_hi), classes of a column consecutive
     * in CSR order with qz descending */
    int32_t cpt, boxz, ncol;
    int32_t a_split;        /* pass A runs bricks of brick[0] / a_split cells in x (more,
                               smaller CTAs: its records are a third of pass B's) */
    const int32_t* bcol_host;
    /* bcmask bit flagging the particles where the restrictphi expression is
     * not skip (its skip pattern depends on x0, y0, z0 only); -1 = evaluate
     * it on every particle */
    int32_t restrict_bit;
    int32_t pad_rb;
    /* opt-in hourglass control (tl_hourglass; no reference counterpart, so no
     * CPU check): pass A writes F into Fh (9 planes) when non-NULL; hg_coef =
     * alpha E / (2 rho0) */
    double hg_coef;
    void* Fh;
    /* time window in which whole-body BC entries can apply: outside it the
     * step treats particles without a BC bit as BC-free */
    double bcw_lo, bcw_hi;
    /* peer-memory halo exchange (multi-GPU slabs, dist.PeerHalo): pass A also
     * stores each boundary particle's pass-B record, and pass B its (u, s)
     * record, straight into the neighbouring ranks' halo rows over NVLink
     * (peer_rb / peer_us: the peers' record arrays, mapped by CUDA IPC).
     * peer_slot: 2 planes of n_all int32, the row of particle i in the side-k
     * peer's arrays, -1 when it is not sent there.  NULL: no peer stores. */
    const int32_t* peer_slot;
    void* peer_us[2];
    void* peer_rb[2];
    /* HOST copy of bcls (ncls entries): the tiled passes take each pair's class
     * geometry (pass B: W, kappa; FP32 2D pass A: W, U) from the constant bank
     * (a kernel parameter) instead of shared memory; NULL keeps the
     * shared-memory table */
    const void* bcls_host;
} tl_body;

#define TL_BRICK_MAX_CLASSES 256
#define TL_BRICK_MAX_COLUMNS 64

/* pass A: F (gated), stress model, history, Laplacian, s-ddot, P L_i and
 * Avis L_i.  Replaces deformation_gradient + update_stress +
 * update_phase_acceleration + np.matmul(F,S) (stepper.py:80-85). */
int tl_pass_a(tl_stream_t st, const tl_body* b);

/* pass B modes */
#define TL_B_INIT 0      /* internal accel + velocity BCs(0,0)   (stepper.py:134-142) */
#define TL_B_VERLET 1    /* + Verlet update                      (stepper.py:144-162) */
#define TL_B_SYMPL 2     /* symplectic corrector                 (stepper.py:176-197) */
/* pass B: momentum + viscosity, a = a_int + f0 + force BCs, velocity BCs,
 * integrator update, phase-field advance + clamps, dt maxima.
 * Replaces momentum + the stepper update phases. */
int tl_pass_b(tl_stream_t st, const tl_body* b, int mode);

/* symplectic predictor (stepper.py:164-175) */
int tl_predict(tl_stream_t st, const tl_body* b);

typedef struct {
    double h, c0;
    unsigned long long* red;   /* the body's dt maxima words (tl_body.red) */
} tl_dtinfo;

/* dt = min(pick_dt, next_out - t, t_max - t) on the device (stepper.py:221-256).
 * When the step proceeds, the maxima words are zeroed after they are read, so
 * the step's pass B accumulates into clean words with no tl_reset_red. */
int tl_clock_begin(tl_stream_t st, tl_clock* clock, int nbody, const tl_dtinfo* info);
/* t += dt, step += 1, output/max_steps halting (stepper.py:199-209, 257-263) */
int tl_clock_commit(tl_stream_t st, tl_clock* clock);
/* reset the dt maxima words of nbody bodies */
int tl_reset_red(tl_stream_t st, unsigned long long* red);
/* deterministic sum of nparts partials into *acc (plastic work) */
int tl_reduce_partials(tl_stream_t st, const double* partials, int64_t nparts, double* acc);

/* Opt-in hourglass control (north star item 6; the reference has none, so
 * it has no CPU check and is off unless requested): the Ganzenmueller (2015)
 * pair force of total-Lagrangian SPH,
 *   f_ij = -(alpha/2) V0_i V0_j W(|X_ij|) E / |X_ij|^2 (d_ij + d_ji) x_ij / |x_ij|,
 *   d_ij = (F_i X_ij - x_ij) . x_ij / |x_ij|,   d_ji with F_j,
 * with X_ij = X_j - X_i and x_ij = x_j - x_i.  It vanishes for an affine
 * deformation and is antisymmetric (momentum conserving).  Adds a_i =
 * sum_j f_ij / m_i into the acceleration planes b->ac (FP64), which pass B
 * adds with the contact term.  Needs the F planes pass A wrote (b->Fh). */
int tl_hourglass(tl_stream_t st, const tl_body* b);

/* Test hook: the fused pass A's FP64 SVK + spectral split (fast.py:224-284
 * semantics, fracture on) on caller-given H = F - I (n x 9, row-major):
 * S (n x 9), psi, psi+ (n); closed[i] = 1 where the closed-form split ran,
 * 0 where it fell back to cyclic Jacobi (near-degenerate spectrum at the
 * sign boundary). */
int tl_svk_split_check(tl_stream_t st, int64_t n, const double* H, double lam, double mu,
                       const double* s, double* S, double* psi, double* psip, int32_t* closed);

/* CTAs of an untiled tl_pass_a (256 particles each); a tiled launch has
 * ceil(n / tile).  pw_partial needs one double per CTA. */
int64_t tl_pass_blocks(int64_t n);

/* ---------------------------------------------------------------------------
 * Output reductions (output.cu).  Per-block FP64
 * partials in block order (deterministic); the caller adds them.
 * ------------------------------------------------------------------------- */
/* blocks (= partial triples) tl_energies writes for n particles */
int64_t tl_energy_blocks(int64_t n);
/* (V0 psi_e, 1/2 m0 |v|^2, V0 Gc [(1-s)^2/(4 eps0) + eps0 |grad s|^2]) partials
 * of the owned particles (output.py:25-49; grad s as backends/fast.py:156-169).
 * Needs the host-layout mirrors (psi_out) of the last output step. */
int tl_energies(tl_stream_t st, const tl_body* b, double* partials);
/* (sum u, sum m0 a) partials, 6 per block of 256, over device positions
 * pos[0..m) (output.py:63-71) */
int tl_measure(tl_stream_t st, const tl_body* b, const int32_t* pos, int64_t m, double* partials);

/* VTK snapshot fields of the owned particles (output.py:84-127 write_vtk_snapshot:
 * current position, displacement, velocity, phase field or equivalent plastic
 * strain, and constitutive.py:154-165 cauchy_batch's stress xx yy zz xy xz yz):
 * 16 doubles per particle at row dst[i] of out, in the caller's order, from
 * the F/S mirrors of the last output step.  One contiguous buffer, for an
 * asynchronous device->host copy that overlaps the next steps. */
int tl_snapshot(tl_stream_t st, const tl_body* b, const int64_t* dst, double* out);

/* ---------------------------------------------------------------------------
 * Penalty contact between two bodies (contact.cu; dynamics.py:81-135,
 * backends/fast.py:426-469).  Current positions x = X + u, velocities v.
 * ------------------------------------------------------------------------- */
typedef struct {
    int64_t n, n_all;       /* owned particles; plane stride */
    int32_t precision;      /* 4 | 8: Real of us / v */
    int32_t uniform;        /* m0 == m0c for every particle */
    double m0c;
    const double* Xs;       /* 3 FP64 planes (device order) */
    const void* us;         /* records (ux uy uz s) */
    const void* v;          /* 3 planes */
    const double* m0;       /* per particle when !uniform */
    const int32_t* perm;    /* device position -> original index (summation order) */
} tl_contact_side;
/* scratch bytes tl_contact_pair needs (cell grid of at most cell_cap cells) */
int tl_contact_workspace_bytes(int64_t n_a, int64_t n_b, int64_t cell_cap, int64_t* bytes);
/* accumulate the contact accelerations of the pair (a, b) into acc_a / acc_b
 * (3 FP64 planes each, stride n_all, NOT cleared): each particle adds its
 * partners' terms in ascending original partner index, the reference's
 * order.  counters[0] += near-coincident pairs (the reference's n_warn),
 * counters[1] += candidates dropped over TL_CONTACT_CAP (must stay 0). */
int tl_contact_pair(tl_stream_t st, const tl_contact_side* a, const tl_contact_side* b, int dim,
                    double dpc, double k_n, double c_n, double kfric, int64_t cell_cap, void* work,
                    int64_t work_bytes, double* acc_a, double* acc_b, unsigned long long* counters);

#ifdef __cplusplus
}
#endif
#endif /* TLSPH_H */
