/*
 * vfmm.h -- C ABI of the B200-native periodic vortex FMM (libvfmm.so).
 *
 * One call, vfmm_evaluate(), computes for N vortex particles in the triply
 * periodic box [lo, lo+len)^3 the regularized Biot-Savart velocity and the
 * vortex-stretching term of Yokota & Barba, arXiv:1110.2921:
 *
 *   u_i        = sum_n sum_j gamma_j x grad(G g_sigma)            PAPER.md:81  Eq.(5)
 *   dgamma_i/dt = sum_n sum_j grad(gamma_j x grad(G g_sigma)) . gamma_i
 *                                                                  PAPER.md:100 Eq.(8)
 *   G = 1/(4 pi r), g_sigma the Gaussian cutoff (Eq. 6),
 *   zeta_sigma the Gaussian core (Eq. 4), n over the periodic image cube
 *   (PAPER.md:164 "3^3 x 3^3 x 3^3 - 1" images; :361 "27^3 periodic images").
 *
 * by the fast multipole method of PAPER.md section 3.1 (Eqs. 10-15):
 * Morton-sorted uniform octree, P2M / M2M, periodic images via multipole
 * expansions, M2L, L2L / L2P (far field without cutoff),
 * and the exact near field P2P ("solving Eq. (5) exactly").
 * Readings of the paper (sign, stretching scheme, image set, ...) are listed in
 * DESIGN.md, section "Readings"; the physical sign u = +curl(psi) is used.
 *
 * Conventions for every function:
 *  - All functions return vfmm_status; nothing throws across the ABI.
 *  - Device buffers are plain CUDA device pointers (cudaMalloc'd or torch-owned);
 *    "host" buffers are ordinary host memory.  The caller owns every buffer it passes.
 *  - Arrays are float32 SoA "3 x n": x[0..n), then y[0..n), then z[0..n).
 *  - A context is bound to one device and is not thread-safe; distinct contexts may
 *    run concurrently on distinct devices.
 */
#ifndef VFMM_H
#define VFMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VFMM_ABI_VERSION 2 /* 2: distributed inputs anywhere in the box; ms_comm fields */
#define VFMM_PMAX 16 /* highest supported expansion order p */

typedef struct vfmm_ctx vfmm_ctx; /* opaque: workspace, operator tables, streams */

typedef enum {
    VFMM_OK = 0,
    VFMM_EINVAL = -1,  /* bad parameter: n < 1, p < 1 or p > VFMM_PMAX, sigma <= 0 or not
                          finite, depth out of [-1, 10], image_levels out of [0, 6], box_len <= 0,
                          NULL pointer, aliasing outputs */
    VFMM_EDOMAIN = -2, /* device-detected (sticky until vfmm_sync_status): a position outside
                          [lo, lo+len)^3 or a non-finite input; outputs are unspecified then */
    VFMM_ENOMEM = -3,  /* device allocation failed */
    VFMM_ECUDA = -4,   /* CUDA runtime error; message in vfmm_last_error_message */
    VFMM_ENCCL = -5,   /* NCCL error (distributed contexts) */
    VFMM_ESTATE = -6   /* call not valid in this state (e.g. debug query before evaluate) */
} vfmm_status;

/* Stretching contraction of Eq. (8) (reading R2 in DESIGN.md). */
typedef enum {
    VFMM_STRETCH_CLASSICAL = 0, /* (gamma_i . grad) u   -- Eq. (2)'s omega . grad u, default */
    VFMM_STRETCH_TRANSPOSE = 1  /* (grad u)^T gamma_i */
} vfmm_scheme;

/* What vfmm_evaluate computes.  DIRECT / NEAR_ONLY / FAR_ONLY exist for tests. */
typedef enum {
    VFMM_MODE_FMM = 0,       /* near (P2P over 27 leaves) + far (expansions)               */
    VFMM_MODE_DIRECT = 1,    /* all-pairs exact sum over the image cube (O(N^2 27^L), tests) */
    VFMM_MODE_NEAR_ONLY = 2, /* only the P2P part of MODE_FMM                               */
    VFMM_MODE_FAR_ONLY = 3,  /* only the expansion part of MODE_FMM                          */
    VFMM_MODE_HYBRID = 4     /* hybrid treecode-FMM auto-tuning: the first
                                evaluate of a new (n, p, image_levels, depth) times the FMM and
                                the treecode (vfmm_evaluate_tree, theta = 0.5) at n_crit = 32,
                                64 and 128, and the context keeps the fastest; not for
                                distributed contexts                                           */
} vfmm_mode;

typedef struct {
    int32_t p;            /* expansion order: degrees n = 0..p, (p+1)^2 coefficients per
                             component (PAPER.md:123 Eq. 10; paper default p = 10, :163)       */
    int32_t depth;        /* uniform octree depth L >= 1: 8^L leaves ("number of
                             levels"); 0 = auto (about 64 particles per leaf); -1 = tuned: the
                             first evaluate of a new n times the auto depth and its two
                             neighbours and keeps the fastest ("automatically choosing the
                             number of particles per box")                    */
    int32_t image_levels; /* 0 = free space; k >= 1: image cube {-m..m}^3, m = (3^k - 1)/2;
                             k = 3 gives the paper's 27^3 boxes           */
    int32_t scheme;       /* vfmm_scheme                                                       */
    int32_t mode;         /* vfmm_mode                                                         */
    float sigma;          /* Gaussian core radius sigma > 0, uniform (Eqs. 4-6)                */
    float box_lo;         /* box is [box_lo, box_lo + box_len)^3, half-open; default -pi       */
    float box_len;        /* default (float)(2 pi) ([-pi, pi]^3)                 */
} vfmm_params;

typedef struct {
    double ms_total, ms_keys, ms_sort, ms_tree, ms_p2m, ms_m2m, ms_m2l, ms_l2l, ms_l2p, ms_p2p;
    int64_t n_p2p_pairs;  /* ordered near-field pairs evaluated (incl. self pairs)        */
    int64_t n_m2l;        /* M2L translations (all levels, incl. periodic far images)      */
    int64_t n_m2m, n_l2l; /* child-parent translations                                     */
    int32_t depth_used;
    int32_t n_kernel_launches; /* kernels launched by the last evaluate                  */
    int64_t bytes_sent, bytes_recv; /* distributed contexts: bytes this rank sent / received
                                       (redistribution both ways, halo particles, LET cells) */
    double ms_comm;         /* distributed contexts: device time of the exchanges (NCCL or
                               logical-rank copies), summed                                  */
    double ms_comm_exposed; /* part of ms_comm the compute stream waited for (not overlapped) */
} vfmm_stats;

/* ABI version this library was built with (VFMM_ABI_VERSION). */
int32_t vfmm_abi_version(void);

/* Fill *prm with defaults: p = 10, depth = 0 (auto), image_levels = 3, classical scheme,
   FMM mode, sigma = 2 pi / 256, box = [(float)-pi, (float)-pi + (float)(2 pi)). */
void vfmm_params_default(vfmm_params* prm);

/* Create a context on CUDA device `device`.  Validates *prm (VFMM_EINVAL, synchronous),
   builds the translation operators once in double precision on the host and uploads them.
   *ctx is set to NULL on failure. */
vfmm_status vfmm_create(vfmm_ctx** ctx, const vfmm_params* prm, int device);

/* Evaluate velocity and stretching for n particles.  Asynchronous on `cuda_stream`
   (a cudaStream_t; NULL = legacy default stream).
     pos    device, 3 x n float32, read-only: positions, already wrapped into the box
     gamma  device, 3 x n float32, read-only: vortex strengths gamma_j (Eq. 3)
     vel    device, 3 x n float32, written:   u_i in input order (Eq. 5)
     dgamma device, 3 x n float32, written:   dgamma_i/dt in input order (Eq. 8)
   Outputs are fully overwritten and must not alias inputs or each other.  The workspace
   grows on the first call with a larger n; steady state performs no allocation.
   Parameter errors return synchronously; input-domain errors are sticky on the device and
   reported by vfmm_sync_status(). */
vfmm_status vfmm_evaluate(vfmm_ctx* ctx, int64_t n, const float* pos, const float* gamma,
                          float* vel, float* dgamma, void* cuda_stream);

/* Velocity at target points that are not particles (NEXT-3: e.g. the velocity on an n^3
   lattice for the energy spectrum): u(t_k) = sum_n sum_j gamma_j x grad(G
   g_sigma)(t_k - x_j - n len) (Eq. 5) from n_src particles (pos, gamma: device,
   3 x n_src) at n_tgt targets (tpos: device, 3 x n_tgt, inside the box) -> tvel (device,
   3 x n_tgt).  The targets join the tree as zero-strength particles (they contribute nothing as
   sources) and take the same near / far path as the particles; the particles' own velocities
   are not returned.  Asynchronous on `cuda_stream`.  Distributed contexts: collective, each rank
   passes its own sources and targets. */
vfmm_status vfmm_evaluate_at(vfmm_ctx* ctx, int64_t n_src, const float* pos, const float* gamma,
                             int64_t n_tgt, const float* tpos, float* tvel, void* cuda_stream);

/* ---- NEXT-4: hybrid treecode, cell-particle traversal (section 3.2) ----
   Velocity and stretching as vfmm_evaluate computes them (Eqs. 5 and 8), by a stack-based
   traversal of an adaptive octree instead of the uniform FMM: the leaves are the non-empty
   cells holding <= n_crit particles (or at the finest level, the context's depth, 0 = auto),
   "automatically choosing the number of particles per box" (reading R22 in
   DESIGN.md).  For each leaf B of targets the traversal starts from the near 3^3 root images
   (free space: the root) and pops cells S: if r_S + r_B < theta |c_B - c_S| (r = half
   diagonal, the multipole acceptance criterion) S acts on every target of B through its
   multipole (cell-particle, M2P: Eq. 11's local expansion of order 2 at the target point,
   then Eqs. 12-15; no cutoff), unless S holds fewer than (p+1)^2 particles,
   when it acts particle-particle (exact and cheaper); else a leaf S acts particle-particle
   (Eq. 5 / Eq. 8 exactly); else its non-empty children are pushed.  Images outside the
   near block come through the root local expansion as in vfmm_evaluate (image_levels >= 2).
   The context's p, depth, image_levels, sigma and scheme apply; its mode is ignored.
   pos, gamma: device 3 x n (SoA), vel, dgamma: device 3 x n outputs (no aliasing), input order.
   theta in [0, 1) (0: every interaction particle-particle, the direct sum over the near
   block), n_crit >= 1; else VFMM_EINVAL.  Not for distributed contexts (VFMM_EINVAL).
   Asynchronous on `cuda_stream`; vfmm_get_stats reports n_p2p_pairs (ordered pairs) and, in
   n_m2l, the number of cell-particle interactions. */
vfmm_status vfmm_evaluate_tree(vfmm_ctx* ctx, int64_t n, const float* pos, const float* gamma,
                               float* vel, float* dgamma, float theta, int32_t n_crit,
                               void* cuda_stream);

/* One forward-Euler time step of the vortex particle method (section 2; forward
   Euler), the three updates simultaneous:
     x_i     += u_i dt          convection, Eq. (7) PAPER.md:91 (wrapped into the box when
                                image_levels > 0; positions stay in [lo, lo+len))
     gamma_i += dgamma_i/dt dt  stretching, Eq. (8)
     sigma^2 += 2 nu dt         diffusion by core spreading, Eq. (9)
   u and dgamma/dt are evaluated as vfmm_evaluate does at the current (x, gamma, sigma)
   and written to vel / dgamma (device, 3 x n, may be NULL); pos and gamma (device, 3 x n) are
   updated in place.  The context's sigma becomes sqrt(sigma^2 + 2 nu dt) (uniform core,
   reading R4) for the next step; *sigma_out (may be NULL) receives it.  Asynchronous on
   `cuda_stream`; dt must be finite, nu >= 0.  Distributed contexts: every rank steps its own
   particles (collective). */
vfmm_status vfmm_step(vfmm_ctx* ctx, int64_t n, float* pos, float* gamma, float dt, float nu,
                      float* vel, float* dgamma, float* sigma_out, void* cuda_stream);

/* ---- NEXT-2: reinitialization by RBF interpolation ----
   Moves the vorticity of n_old particles (pos_old, gamma_old: device 3 x n_old, core radius
   sigma_old, typically grown by core spreading) onto n_new new particles (pos_new: device
   3 x n_new, usually the cell-centre lattice) of core radius sigma_new (= h):
     omega_i = sum_j gamma_j zeta_sigma_old(x_i - x_j)                  Eq. (3) at the new points
     solve     sum_j gamma'_j zeta_sigma_new(x_i - x_j) = omega_i  for gamma'
   by GMRES(restart) in matrix-free form, the Gaussian sums over neighbour leaves only
   (reading R18: neighbour radius ws with ws a >= 6 sigma, truncation < 1.5e-8),
   initial guess gamma' = omega dx^3 with dx^3 = box_len^3 / n_new, exit when the residual has
   dropped by `tol` relative to that guess's residual, per strength component,
   or after max_iter iterations.  Outputs (device, 3 x n_new, input order of pos_new):
   gamma_new (required), omega_new (may be NULL).  Uses the context's box, image_levels (> 0:
   periodic neighbours) and depth (0 = auto for n_new); sets the context's sigma to sigma_new.
   Synchronous (the GMRES recurrences run on the host); all vector work on `cuda_stream`. */
typedef struct {
    int32_t iterations;      /* GMRES iterations (matrix-vector products after the residual) */
    int32_t converged;       /* 1 if every component reached tol                            */
    double rel_residual[3];  /* final ||omega - A gamma'|| / ||omega - A gamma'_0|| per comp.  */
    double ms;               /* device time of the whole reinitialization                    */
    int32_t depth_used, ws_old, ws_new;
} vfmm_reinit_info;

vfmm_status vfmm_reinit(vfmm_ctx* ctx, int64_t n_old, const float* pos_old,
                        const float* gamma_old, float sigma_old, int64_t n_new,
                        const float* pos_new, float sigma_new, float tol, int32_t max_iter,
                        int32_t restart, float* gamma_new, float* omega_new,
                        vfmm_reinit_info* info, void* cuda_stream);

/* Per-particle core radius (NEXT-4): as vfmm_evaluate, with sigma_j of every particle (device,
   n floats > 0, input order) in the cutoff of Eq. (6) -- PAPER.md:86 writes the source's
   sigma_j -- for the near field (P2P) and DIRECT mode; the far field drops the cutoff
    as before.  The context's sigma must be >= max sigma_j: the automatic depth
   keeps the leaf width >= 4 sigma with it (reading R3).  Single-GPU contexts only. */
vfmm_status vfmm_evaluate_sigma(vfmm_ctx* ctx, int64_t n, const float* pos, const float* gamma,
                                const float* sigma, float* vel, float* dgamma, void* cuda_stream);

/* ---- multi-GPU: Morton-range spatial decomposition + local-essential-tree exchange ----
   (the paper's multi-GPU runs.)  Rank r of R
   (R in {1, 2, 4, 8}) owns the Morton leaf range [r 8^L/R, (r+1) 8^L/R) at depth L
   (vfmm_partition).  Every rank passes its own n (possibly different, possibly 0) particles
   ANYWHERE in the box and gets u, dgamma for them in its own input order: the library
   redistributes them to their owners and returns the results (device-side Morton sort + grouped
   NCCL send/recv both ways).  The result equals a single-context evaluation of the rank-order
   concatenation of all ranks' inputs (same per-target summation order; the tensor-core M2L's
   per-rank f16 staging scale can change the last bits).  depth must be set explicitly (>= 2).
   Halo particles and LET multipoles travel over NCCL on a communication stream that overlaps
   the upward pass and the M2L; two host syncs per evaluation read message sizes. */

/* Write a fresh NCCL unique id (128 bytes) to host memory `out128` (call on one rank and
   broadcast it, e.g. with torch.distributed).  VFMM_ENCCL if libnccl.so.2 is unavailable. */
vfmm_status vfmm_nccl_get_unique_id(void* out128);

/* Collective: create a context for rank `rank` of `nranks` on `device`, initialising an NCCL
   communicator from `nccl_id128` (host, 128 bytes).  prm->depth must be >= 2.  Such a context
   always runs the distributed phases, also for nranks = 1 (a one-rank communicator). */
vfmm_status vfmm_create_nccl(vfmm_ctx** ctx, const vfmm_params* prm, int device,
                             const void* nccl_id128, int nranks, int rank);

/* Owned Morton leaf range [*leaf_lo, *leaf_hi) of `rank` for depth L and `nranks` ranks
   (host helper for partitioning inputs).  VFMM_EINVAL unless nranks in {1,2,4,8}. */
vfmm_status vfmm_partition(int depth, int nranks, int rank, int64_t* leaf_lo, int64_t* leaf_hi);

/* Test mode: run the distributed algorithm for `nranks` LOGICAL ranks on this context's one
   GPU -- every phase of every rank in lockstep, exchanges as device-to-device copies -- so
   the redistribution / partition / halo / LET logic can be validated on a single GPU.  Arrays
   are per rank: n[r] >= 0 particles anywhere in the box at device pointers pos[r], gamma[r],
   results to vel[r], dgamma[r] in rank r's input order.  Synchronizes `cuda_stream`. */
vfmm_status vfmm_evaluate_logical(vfmm_ctx* ctx, int nranks, const int64_t* n,
                                  const float* const* pos, const float* const* gamma,
                                  float* const* vel, float* const* dgamma, void* cuda_stream);

/* Host-only routing of the redistribution (no GPU needed): for n HOST positions (3 x n SoA
   float32, anywhere in [lo, lo+len)^3) write counts[q] = how many fall in rank q's Morton range
   at depth L (q < nranks) -- the send counts this rank's evaluate uses.  VFMM_EDOMAIN if a
   position lies outside the box (the counts are then still written, clamped). */
vfmm_status vfmm_route_counts(int depth, int nranks, int64_t n, const float* pos_h, float box_lo,
                              float box_len, int64_t* counts);

/* Host-only introspection of the static exchange plan of `rank` (no GPU needed): kind 0 =
   halo particle leaves (depth level), kind k in [2, depth] = LET multipole cells of level k;
   dir 0 = ids this rank receives from `peer`, dir 1 = ids it sends to `peer`.  Writes up to
   `cap` ids (ascending Morton index) to `out` (may be NULL) and the full count to *count. */
vfmm_status vfmm_dist_plan(int depth, int nranks, int rank, int periodic, int kind, int dir,
                           int peer, int32_t* out, int64_t cap, int64_t* count);

/* Same as vfmm_evaluate but every buffer is HOST memory (pinned or pageable): copies in,
   evaluates on the context's internal stream, copies out, synchronizes. */
vfmm_status vfmm_evaluate_host(vfmm_ctx* ctx, int64_t n, const float* pos_h,
                               const float* gamma_h, float* vel_h, float* dgamma_h);

/* Synchronize the last evaluate's stream; return VFMM_EDOMAIN if the device flagged bad
   input (and clear the flag), else VFMM_OK or a CUDA error. */
vfmm_status vfmm_sync_status(vfmm_ctx* ctx);

/* Per-phase timings (CUDA events) and counters of the last evaluate; synchronizes. */
vfmm_status vfmm_get_stats(vfmm_ctx* ctx, vfmm_stats* out);

/* Change p / depth / image_levels / scheme / mode / sigma / box of an existing context
   (rebuilds operator tables if p changed).  Synchronous. */
vfmm_status vfmm_set_params(vfmm_ctx* ctx, const vfmm_params* prm);

/* Tree of the last evaluate, copied to HOST buffers (synchronizes):
   keys_sorted, perm: n entries (uint32); leaf_start: 8^depth + 1 entries (int32).
   perm[k] = input index of the k-th particle in Morton order (stable sort);
   leaf_start[c] = number of keys < c.  Any pointer may be NULL. */
vfmm_status vfmm_debug_tree(vfmm_ctx* ctx, uint32_t* keys_sorted, uint32_t* perm,
                            int32_t* leaf_start);

/* Expansion coefficients of the last FMM evaluate at tree level `level` (0..depth),
   copied to HOST (synchronizes).  kind 0 = multipole, 1 = local.  Layout:
   [cell (Morton index at that level)][component x,y,z][(p+1)^2] float32, packed real form
   of DESIGN.md "Expansion convention" (index n^2 for Re(n,0); n^2+2m-1, n^2+2m for
   Re, Im of (n, m>0)), normalised by the cell width a_l: multipole / a^n, local * a^(n+1).
   `out` must hold 8^level * 3 * (p+1)^2 floats. */
vfmm_status vfmm_debug_expansions(vfmm_ctx* ctx, int kind, int level, float* out);

/* Human-readable status name, and the last detailed error message of a context. */
const char* vfmm_strerror(vfmm_status s);
const char* vfmm_last_error_message(const vfmm_ctx* ctx);

/* Release the context and everything it owns.  NULL is a no-op. */
void vfmm_destroy(vfmm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* VFMM_H */
