/*
 * include/odp.h -- C-ABI of the B200-native time-dependent Hamilton-Jacobi level-set step
 * (OptimizedDP, Bui et al., arXiv 2204.05520).  Implemented by paper_2204_05520_b200/libodp.so
 * (hand-written sm_100a CUDA kernels + a C++ host orchestrator).
 *
 * What the library computes (§3.2, Eq. 4):
 *     D_s phi(z,s) + H(z, grad phi) = 0,  H = min_d max_u grad(phi)^T f(z,u,d),  phi(z,0) = phi0(z)
 * solved backward in time (tau = -s >= 0, V_tau = H) by the level-set algorithm of Algorithm 2
 * (P:146-172): per node one-sided derivatives (§3.4.4), optimal control/disturbance and
 * Hamiltonian (l.153-156), global derivative range (l.157-158), Lax-Friedrichs dissipation with
 * alpha_i (l.160-164, dissipation sign per DESIGN.md reading A2), CFL time step (l.167, §3.4.3
 * P:243), Runge-Kutta update (l.169); BRT = min with the target after every full step (reading
 * A11).  The grid follows §3.4.1.  Every reading of the paper is listed in DESIGN.md §3.
 *
 * Conventions for every function:
 *   - returns odp_status; never throws across the ABI; on failure odp_last_error() holds a
 *     message (thread-local, valid until the next call from the same thread);
 *   - arrays are row-major with axis 0 outermost and axis dims-1 contiguous (§4.1);
 *   - value arrays are float32; coordinates, bounds, params and times are float64.
 */
#ifndef ODP_H_
#define ODP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ODP_OK = 0,
    ODP_EINVAL = 1,    /* argument validation failed (before any device work)              */
    ODP_ENUMERIC = 2,  /* NaN or max|V| > 1e10 in a stage input (reading A19)   */
    ODP_ECUDA = 3,     /* a CUDA runtime call or kernel launch failed                       */
    ODP_ENCCL = 4,     /* an NCCL call of the multi-GPU transport failed (or NCCL missing)   */
    ODP_ENOMEM = 5     /* device or host allocation failed                                   */
} odp_status;

typedef enum {
    ODP_LOW = 1,       /* first-order upwind derivatives + forward Euler (stencil radius 1)  */
    ODP_MEDIUM = 2     /* second-order ENO derivatives + TVD-RK2 (Heun)  (stencil radius 2)  */
} odp_accuracy;

typedef enum { ODP_BRS = 0, ODP_BRT = 1 } odp_mode;

/* Compiled-in dynamics.  params layouts (doubles); goal = -1 to
 * minimise (reach), +1 to maximise (avoid); the disturbance always takes the opposite goal:
 *   HOLONOMIC_BALL [ubar, goal]                xdot = u, |u|_2 <= ubar          (any dims)
 *   HOLONOMIC_BOX  [ubar, dbar, goal]          xdot_i = u_i + d_i              (any dims)
 *   DUBINS3D       [v, wbar, goal]             (x, y, th): v cos th, v sin th, w
 *   CAR4D          [abar, wbar, dxbar, dybar, goal]  (x, y, v, th): v cos th + dx, v sin th + dy, a, w
 *   CAR5D          [abar, alphabar, goal]      (x, y, th, v, w): v cos th, v sin th, w, a, alpha
 *   DOUBLEINT6D    [ubar, dbar, goal]          (px, vx, py, vy, pz, vz): v_i, u_i + d_i
 *   PAIR_DUBINS3D  [va, vb, abar, bbar, goal]  (x, y, th): -va + vb cos th + a y, va sin th - a x, b - a;
 *                  a (evader) takes the goal's extremum, b (pursuer) the opposite (reading A30) */
typedef enum {
    ODP_DYN_HOLONOMIC_BALL = 0,
    ODP_DYN_HOLONOMIC_BOX = 1,
    ODP_DYN_DUBINS3D = 2,
    ODP_DYN_CAR4D = 3,
    ODP_DYN_CAR5D = 4,
    ODP_DYN_DOUBLEINT6D = 5,
    ODP_DYN_PAIR_DUBINS3D = 6   /* Eq. 7, the paper's own 3D example */
} odp_dynamics;

/* Kernel family used for the two passes of every stage. */
typedef enum {
    ODP_KERNEL_AUTO = 0,     /* resident on small grids (below), else march, else stream, else
                                tiled, else generic -- the first that covers the grid          */
    ODP_KERNEL_GENERIC = 1,  /* one thread per node, neighbours through L1/L2                 */
    ODP_KERNEL_TILED = 2,    /* inner-plane tile + every outer neighbour tile staged in shared
                                memory by 1-D TMA bulk copies (mbarrier pipeline)             */
    ODP_KERNEL_STREAM = 3,   /* CTA marches the innermost outer axis with a register window;
                                in-plane tile in padded shared memory                          */
    ODP_KERNEL_MARCH = 4,    /* the stream decomposition with edge-shared ENO2 picks carried
                                along the marching axis, edge-assigned pass 1, packed FP32x2
                                arithmetic and one barrier per step (kernels_march.cuh)       */
    ODP_KERNEL_RESIDENT = 5  /* small grids: the WHOLE solve (every interval, step, stage,
                                finalize and snapshot) in one cooperative launch with grid
                                barriers between the passes; the generic per-node arithmetic
                                (bitwise the generic family's result).  AUTO picks it on one
                                rank for grids up to 2^18 nodes (env ODP_RESIDENT_MAX_POINTS)
                                unless kernel_ms or single_pass is requested.  Not for
                                PAIR_DUBINS3D (alpha^max over three axes).  ODP_EINVAL when
                                requested where it does not apply.                             */
} odp_kernel;

typedef struct odp_grid odp_grid;   /* opaque; one solve at a time per handle */

typedef struct {
    double cfl;               /* CFL factor C; <= 0 selects the default 0.8 (LOW) / 0.5 (MEDIUM) (A7) */
    const float *target;      /* BRT min operand (device, same layout as V0); NULL -> V0.  Separate
                                 from V0 so a solve can restart from a snapshot    */
    void *stream;             /* cudaStream_t to run on; NULL -> the library's own stream          */
    int write_initial;        /* 1 -> out holds ntau slices, out[0] = V0; 0 -> ntau-1 slices       */
    int kernel;               /* odp_kernel                                                         */
    int use_graph;            /* 1 -> replay the per-step launch sequence as a CUDA graph          */
    double *tau_reached;      /* optional out: tau at return (valid on ODP_ENUMERIC too)            */
    long long *steps_taken;   /* optional out: time steps taken                                     */
    long long *stages_taken;  /* optional out: RK stages evaluated                                  */
    double *kernel_ms;        /* optional out [4]: summed device time of pass 1, pass 2, finalize,  *
                               * and of the pass-2 launches of RK stage 2 (included in [1])          */
    int single_pass;          /* 1 -> SURVEY.md §8(f1): when the functor's alpha does not depend on
                                 the derivative range (HOLONOMIC_BOX, DUBINS3D, CAR5D, DOUBLEINT6D)
                                 and the march kernels cover the grid, skip pass 1 after the first
                                 step: alpha^max is fixed, dt is re-derived from it, and the guard
                                 (NaN, |V| > 1e10) checks every stage's output.  Bitwise the
                                 two-pass result.  0 (default) -> Algorithm 2's two passes        */
    int *single_pass_used;    /* optional out: 1 if the single-pass path ran                      */
} odp_solve_opts;

/*
 * odp_grid_create -- Cartesian grid of §3.4.1: node counts N[d], bounds [lo[d], hi[d]]
 * and a periodic bit per axis (bit d of periodic_mask).  Spacing (hi-lo)/(N-1), or (hi-lo)/N on
 * periodic axes whose upper endpoint is excluded (reading A15).  Host pointers, copied.
 * Errors: ODP_EINVAL if dims is not in 1..6, any N[d] < 3, or lo[d] >= hi[d].
 * Ownership: the caller destroys the handle with odp_grid_destroy.
 */
odp_status odp_grid_create(int dims, const double *lo, const double *hi, const int64_t *N,
                           uint32_t periodic_mask, odp_grid **out);

/* Frees the handle and the device working buffers it caches.  NULL is ignored. */
void odp_grid_destroy(odp_grid *g);

/* Copies dims, the global N[0..dims), the spacing dx[0..dims) and the point count of the handle's
 * (local) grid -- the whole grid unless partitioned (any out pointer may be NULL). */
odp_status odp_grid_info(const odp_grid *g, int *dims, int64_t *N, double *dx, int64_t *points);

/*
 * odp_hj_solve -- solve Eq. 4 from V0 through the save times tau[0..ntau) (tau[0] = 0, strictly
 * increasing, float64 host array) on the current CUDA device.
 *   dynamics_id, params, nparams  a compiled-in functor and its parameters (host doubles)
 *   V0       DEVICE pointer, points() float32 values: phi0 on the nodes (initial value and, unless
 *            opts->target is given, the BRT target)
 *   accuracy ODP_LOW | ODP_MEDIUM;  mode ODP_BRS | ODP_BRT
 *   out      DEVICE pointer, (ntau-1) x points() floats (ntau x points() with write_initial):
 *            out[k] = V(tau[k+1]).  Must not alias V0.
 *   opts     nullable.
 * Ownership: caller owns V0, out, params, tau, target; the library owns its working buffers.
 * Errors: ODP_EINVAL (bad ids, param count, dims mismatch with the functor, ntau < 2, tau[0] != 0,
 * unsorted tau, NULL pointers); ODP_ENUMERIC (NaN or |V| > 1e10 in a stage input -- snapshots up
 * to the last completed save time are valid and tau_reached is set); ODP_ECUDA; ODP_ENOMEM.
 * The call returns after the device work has completed (it synchronises its stream).
 */
odp_status odp_hj_solve(odp_grid *g, int dynamics_id, const double *params, int nparams,
                        const float *V0, const double *tau, int ntau, int accuracy, int mode,
                        float *out, const odp_solve_opts *opts);

/*
 * odp_hj_solve_host -- as odp_hj_solve, but V0, out and opts->target are HOST pointers.  The
 * library allocates device copies, copies V0 (and target) in, solves, and copies every snapshot
 * back to `out` before returning (the end-to-end path; pinned host memory is fastest).
 */
odp_status odp_hj_solve_host(odp_grid *g, int dynamics_id, const double *params, int nparams,
                             const float *V0, const double *tau, int ntau, int accuracy, int mode,
                             float *out, const odp_solve_opts *opts);

/*
 * Multi-GPU: axis-0 slab partition (north_star: "Large grids are slab-partitioned along axis 0 ...
 * Each RK stage does an NCCL send/recv halo exchange over NVLink, and an allreduce-max of alpha per
 * step"; the method's per-node independence within a stage, §4.2).
 *
 * odp_partition_extent -- the slab of `rank` among `nranks` over N0 axis-0 planes: contiguous,
 *   balanced (the first N0 mod nranks ranks own one plane more).  Pure host arithmetic.
 * odp_comm_unique_id -- writes a 128-byte NCCL unique id (call on rank 0; the caller broadcasts
 *   it, e.g. with torch.distributed).  NCCL is loaded on first use (libnccl.so.2); ODP_ENCCL if it
 *   cannot be loaded.
 * odp_grid_partition -- makes the handle describe rank `rank`'s slab and joins the NCCL
 *   communicator (collective: every rank calls it with the same id).  `device` is the CUDA device of
 *   this rank.  After it, odp_hj_solve / odp_hj_solve_host take V0, out and target as LOCAL slab
 *   arrays (i0_count x prod_{d>=1} N[d] floats, row-major), odp_grid_info reports the global N and
 *   the local point count, and every stage exchanges R halo planes with the axis-0 neighbours and
 *   allreduces the derivative range, so all ranks take the same dt sequence and the result is
 *   bitwise the one of the unpartitioned solve.  Errors: ODP_EINVAL (rank out of range, a periodic
 *   axis 0, fewer than 2 planes per rank, NULL id with nranks > 1), ODP_ENCCL.  nranks = 1 restores
 *   the whole grid (with an id: a 1-rank communicator, i.e. the multi-GPU code path on one GPU).
 * odp_grid_local_extent -- the slab of this handle: first owned axis-0 plane and the plane count.
 */
odp_status odp_partition_extent(int64_t N0, int nranks, int rank, int64_t *i0_begin, int64_t *i0_count);
odp_status odp_comm_unique_id(void *id128);
odp_status odp_grid_partition(odp_grid *g, int rank, int nranks, const void *id128, int device);
odp_status odp_grid_local_extent(const odp_grid *g, int64_t *i0_begin, int64_t *i0_count);

/*
 * Loopback transport (tests of the multi-rank path with one GPU).  The same slab partition as
 * odp_grid_partition, but the nranks handles live in ONE process on ONE device, each driven by its
 * own host thread: halo planes move by device-to-device copies and the range records are reduced by
 * a max kernel, ordered with stream events and a host barrier per collective (every rank calls the
 * same collectives in the same order -- the property the NCCL path relies on as well).  No kernel
 * waits on another rank's kernel, so the handles' solves never deadlock the device.
 *
 * odp_loopback_create -- a transport for nranks (1..64) handles; *out owned by the caller.
 *   ODP_EINVAL, ODP_ENOMEM, ODP_ECUDA (events, the record buffer on the current device).
 * odp_grid_partition_loopback -- makes `g` rank `rank`'s slab on the transport (the transport must
 *   outlive the handle's solves).  Errors as odp_grid_partition.
 * odp_loopback_destroy -- frees the transport (after every handle on it is destroyed or
 *   re-partitioned).
 */
typedef struct odp_loopback odp_loopback;
odp_status odp_loopback_create(int nranks, odp_loopback **out);
odp_status odp_grid_partition_loopback(odp_grid *g, int rank, odp_loopback *lb);
void odp_loopback_destroy(odp_loopback *lb);

/*
 * Time-to-reach: the stationary HJ equation of Eq. 6 for the TTR
 * function phi(z) = min time to reach the target T = {V0 <= 0} (Eq. 5), by the
 * Lax-Friedrichs iteration of Algorithm 3: phi = 0 on T and `big` elsewhere (l.1);
 * every node not on a non-periodic face takes
 *     phi_new = min(phi, (-H + sum_d sigma_d (phi_{+d} + phi_{-d}) / (2 dz_d)) / (sum_d sigma_d / dz_d))
 * with p = central differences, H = -H_reach(z, p) - 1 (the functor's Hamiltonian with goal -1,
 * whatever params[last] says; it must still be -1 or +1) and sigma_d the functor's alpha on the
 * costate box [-1, 1]^n (readings A32, A33); then along each non-periodic axis in order the faces
 * take min(max(2 phi_1 - phi_2, phi_2), phi_face) (l.14-15, A34); repeat while
 * max |phi - phi_old| > eps (A31).  The GPU iterates in Jacobi order (A35): every node of
 * iteration k+1 from iteration k -- Algorithm 3's fixed point without its sequential dependence.
 *
 *   V0   DEVICE pointer, points() floats: the target is {V0 <= 0}
 *   phi  DEVICE pointer, points() floats: the result (float32).  Must not alias V0.
 *   opts nullable.
 * Errors: ODP_EINVAL (bad dynamics/params as odp_hj_solve, a non-periodic axis with N < 4, a
 * partitioned handle, NULL pointers); ODP_ECUDA; ODP_ENOMEM.  Returns after the device work.
 * Iterations stop at max_iters even if the change is still above eps (iters_taken says so).
 */
typedef struct {
    double eps;               /* stop once max |phi - phi_old| <= eps; <= 0 -> 1e-6 (A31)        */
    long long max_iters;      /* <= 0 -> 100000                                                  */
    double big;               /* initial value off the target; <= 0 -> 100 (l.1)                 */
    void *stream;             /* cudaStream_t; NULL -> the library's own stream                  */
    int use_graph;            /* 1 -> replay chunks of iterations as a CUDA graph                */
    long long *iters_taken;   /* optional out: iterations executed                               */
    double *last_change;      /* optional out: max |phi - phi_old| of the last iteration         */
    double *kernel_ms;        /* optional out [3]: device time of the iteration loop; with
                                 use_graph = 0 also the summed time of the interior launches [1]
                                 and of the face launches [2] of the iterations that ran (per-launch
                                 events), else -1                                                 */
} odp_ttr_opts;

odp_status odp_ttr_solve(odp_grid *g, int dynamics_id, const double *params, int nparams,
                         const float *V0, float *phi, const odp_ttr_opts *opts);

/* As odp_ttr_solve with HOST V0 and phi (copies inside the call). */
odp_status odp_ttr_solve_host(odp_grid *g, int dynamics_id, const double *params, int nparams,
                              const float *V0, float *phi, const odp_ttr_opts *opts);

/*
 * Value iteration: Algorithm 1 for a continuous-state MDP
 * (Eq. 1-3) discretised on the grid's nodes (readings A36-A38):
 *     V_0 = 0;  V_{t+1}(s) = max_a [ R(s) + gamma sum_k p_k V_t(s'_k) ]
 * until max_s |V_{t+1} - V_t| < threshold; s'_k = the node nearest to s + Delta(s, a, k), per
 * axis i + rint(Delta_d / dx_d) in float32, wrapped on periodic axes, clamped on the others.
 * Models (params, doubles):
 *   ODP_MDP_HOLONOMIC [speed, dt, gamma]   any dims; actions {stay, +-e_d}, Delta = +-dt speed e_d
 *   ODP_MDP_DUBINS3D  [vbar, wbar, dt, slip, pslip, gamma]   (x, y, th), th periodic by the caller;
 *       actions v in {vbar/2, vbar} x w in {-wbar, 0, wbar}; outcomes sigma in {0, +slip, -slip}
 *       with probabilities {1 - 2 pslip, pslip, pslip};
 *       Delta = (dt v cos th - sigma sin th, dt v sin th + sigma cos th, dt w)
 *   R  DEVICE pointer, points() floats: the reward of each node (A37)
 *   V  DEVICE pointer, points() floats: the result (float32, Jacobi order).  Must not alias R.
 * Errors: ODP_EINVAL (unknown model, param count, dims, gamma not in [0, 1), pslip not in
 * [0, 0.5], partitioned handle, NULL pointers); ODP_ECUDA; ODP_ENOMEM.  Returns after the device work.
 */
typedef enum { ODP_MDP_HOLONOMIC = 0, ODP_MDP_DUBINS3D = 1 } odp_mdp_model;

typedef struct {
    double threshold;         /* stop after the first iteration with change < threshold; <= 0 -> 1e-6 */
    long long max_iters;      /* <= 0 -> 100000                                                  */
    int fixed_iters;          /* 1 -> ignore the threshold: run exactly max_iters iterations      */
    void *stream;             /* cudaStream_t; NULL -> the library's own stream                  */
    int use_graph;            /* 1 -> replay chunks of iterations as a CUDA graph                */
    long long *iters_taken;   /* optional out: iterations executed                               */
    double *last_change;      /* optional out: max |V_{t+1} - V_t| of the last iteration          */
    double *kernel_ms;        /* optional out [2]: device time of the iteration loop; with
                                 use_graph = 0 also the summed time of the iteration launches [1],
                                 else -1                                                          */
} odp_vi_opts;

odp_status odp_vi_solve(odp_grid *g, int model_id, const double *params, int nparams,
                        const float *R, float *V, const odp_vi_opts *opts);

/* As odp_vi_solve with HOST R and V (copies inside the call). */
odp_status odp_vi_solve_host(odp_grid *g, int model_id, const double *params, int nparams,
                             const float *R, float *V, const odp_vi_opts *opts);

/* Number of kernel launches issued by the last solve on this handle (launch accounting). */
long long odp_last_launch_count(const odp_grid *g);

/* Human-readable message for the last failing call on this thread ("" if none). */
const char *odp_last_error(void);

/* Library version string, e.g. "odp-b200 0.1 sm_100a". */
const char *odp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ODP_H_ */
