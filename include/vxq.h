/*
 * vxq.h -- C-ABI of the B200-native batched multi-replica dynamics loop.
 *
 * This is the drop-in boundary for the reference's hot path
 * (qubokit, /root/reference/pkg/src/qubokit):
 *
 *   reference entry point                              replaced by
 *   -------------------------------------------------  ------------------------------
 *   IsingModel + coupling_operator()/_csr              vxq_problem_create
 *       model.py:113-192 (frozen COO i<j, h, offset)
 *   solve_pa(model, PaParams) -> SampleSet             vxq_pa_solve
 *       solvers/parallel_annealing.py:28-48
 *   solve_sbm(model, SbmParams) -> SampleSet           vxq_sbm_solve
 *       solvers/bifurcation.py:50-67
 *   integrate(B, g, Q, P, dt, a_schedule, a0, c0, q)   vxq_sbm_integrate
 *       solvers/bifurcation.py:37-47
 *   solve_sa(model, SaParams) -> SampleSet             vxq_sa_solve
 *       solvers/annealing.py:24-74
 *   IsingModel.energies(states)                        vxq_energies
 *       model.py:160-164 (here: correctly rounded exact sums)
 *   resolve_lambda0 / field_scale                      vxq_problem_lambda0
 *       parallel_annealing.py:23-25, model.py:194-200
 *   resolve_c0 / eig_extreme(-A, "max")                vxq_problem_c0
 *       bifurcation.py:25-34, solvers/eigen.py:35-56
 *
 * Conventions: plain host pointers and sizes; no torch types.  All entry
 * points are reentrant (one CUDA stream + stream-ordered workspace per call,
 * no global mutable state beyond a per-device context cache).  Return 0 on
 * success, else a VXQ_ERR_* code; vxq_last_error() gives a thread-local
 * message.  Parameter validation (ValidationError in the reference,
 * common.py:109-116,136-144) happens in the host layer before the call; the
 * C layer re-checks and returns VXQ_ERR_INVALID.
 */
#ifndef VXQ_H_
#define VXQ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define VXQ_API __attribute__((visibility("default")))
#else
#define VXQ_API
#endif

#define VXQ_ABI_VERSION 5  /* 5: outputs.step_kernel; 4: eig_info, dense_eligible, outputs.dense_kind, session snapshots */

#define VXQ_OK 0
#define VXQ_ERR_INVALID 1     /* -> ValidationError */
#define VXQ_ERR_OOM 2         /* -> QubokitError    */
#define VXQ_ERR_CUDA 3        /* -> QubokitError    */
#define VXQ_ERR_UNSUPPORTED 4 /* -> QubokitError    */

/* precision of the dynamics loop */
#define VXQ_FP32 0 /* default: fp32 state, fp32 CSR values, sequential row sums */
#define VXQ_FP64 1 /* parity mode: bit-exact with the reference's CSR path     */

/* kernel path */
#define VXQ_PATH_AUTO 0
#define VXQ_PATH_RESIDENT 1 /* small n: one CTA owns replicas for all T steps  */
#define VXQ_PATH_SPARSE 2   /* CSR SpMM + fused integrator, one launch per step */
#define VXQ_PATH_DENSE 3    /* tcgen05/TMEM J.S GEMM with fused integrator      */

typedef struct vxq_problem vxq_problem;

/* PaParams (common.py:94-116). lambda0 NaN => auto (field scale). */
typedef struct {
    int64_t steps;
    double learning_rate;
    double momentum;
    double lambda0;
    int64_t replicas;
    uint64_t seed;
} vxq_pa_params;

/* SbmParams (common.py:119-144). c0 NaN => auto (1 / lambda_max(-A)). */
typedef struct {
    int64_t steps;
    double dt;
    double a0;
    double c0;
    double q_cap;
    double init_noise;
    int64_t replicas;
    uint64_t seed;
} vxq_sbm_params;

/* SaParams (common.py:74-92), geometric schedule.  T_init NaN => 2 * max(field_scale,
 * 1e-12); T_final NaN => 1e-3 * T_init (annealing.py:29-30).  temps: optional HOST array
 * [sweeps], the temperature of each sweep; the Python layer passes numpy's
 * T_init * ratio ** arange(sweeps) so it is bit-identical with annealing.py:31-35
 * (NULL => vxq_sa_schedule, C pow). */
typedef struct {
    int64_t sweeps;
    double T_init;
    double T_final;
    int64_t replicas;
    uint64_t seed;
    const double* temps;
} vxq_sa_params;

typedef struct {
    int32_t precision;         /* VXQ_FP32 | VXQ_FP64                            */
    int32_t path;              /* VXQ_PATH_*                                     */
    int32_t outputs_on_device; /* 1: vxq_outputs pointers are device pointers    */
    int32_t track_best;        /* 1: states/energies = best state seen per replica
                                  (over s_0..s_T; sparse/resident paths; opt-in)   */
    int64_t replica_begin;     /* global index of local replica 0 (sharding)     */
    void* stream;              /* cudaStream_t; NULL => library stream (pass
                                  cudaStreamLegacy, (void*)1, for the legacy default) */
} vxq_run_opts;

typedef struct {
    int8_t* states;      /* [R][n] spins (+1/-1), replica-major  (required) */
    double* energies;    /* [R] exact energies                    (required) */
    double* x;           /* [R][n] final X (PA) / Q (SBM), optional          */
    double* m;           /* [R][n] final M (PA) / P (SBM), optional          */
    int64_t* order;      /* [R] replicas by ascending energy, ties by index (optional;
                            argsort(kind="stable") of common.py:57)                  */
    double* energy_trace; /* [T] optional: min over replicas of E(s_t), the energy of
                             the spins entering step t (exact on the sparse paths and on
                             the dense uniform-|J| paths with h = 0 -- PA fused, SBM via
                             a spin plane next to the digit planes; NaN on the general-J
                             dense SBM) -> time-to-target                               */
    /* filled by the library */
    double lambda0_used; /* PA: lambda0;  SA: T_init  */
    double c0_used;      /* SBM: c0;      SA: T_final */
    double loop_ms;      /* device time of the dynamics loop (CUDA events)   */
    int64_t launches;    /* kernels launched by this call                    */
    int32_t path_used;   /* VXQ_PATH_* actually run                          */
    int32_t dense_kind;  /* VXQ_DENSE_KIND_*: operand scheme of the tensor-core path */
    int32_t step_kernel; /* VXQ_KERNEL_*: the dynamics kernel that ran (ABI 5)       */
    int32_t reserved;
} vxq_outputs;

/* dynamics kernels (vxq_outputs.step_kernel) */
#define VXQ_KERNEL_NONE 0
#define VXQ_KERNEL_PA_STEP 1       /* CSR step over bit-packed spins, one launch per step  */
#define VXQ_KERNEL_PA_STEP_COOP 2  /* the same for R <= 32 (8 rows per warp)               */
#define VXQ_KERNEL_PA_CLUSTER 3    /* thread-block clusters, spin tables in shared memory   */
#define VXQ_KERNEL_PA_RESIDENT 4   /* small n: state + CSR in shared memory, one launch     */
#define VXQ_KERNEL_SBM_STEP 5      /* CSR step over fp32/fp64 q, one launch per step        */
#define VXQ_KERNEL_SBM_BLOCK 6     /* row blocks: distinct neighbours' q staged in smem     */
#define VXQ_KERNEL_SBM_RESIDENT 7
#define VXQ_KERNEL_DENSE_RUN 8     /* tcgen05 persistent dense kernel (see dense_kind)      */
#define VXQ_KERNEL_SA_RUN 9

/* tensor-core operand schemes (vxq_outputs.dense_kind) */
#define VXQ_DENSE_KIND_NONE 0
#define VXQ_DENSE_KIND_MXF4 1    /* PA, uniform |J|: K, spins packed E2M1, kind::mxf4       */
#define VXQ_DENSE_KIND_F8F6F4 2  /* PA, uniform |J|: kind::f8f6f4 (VXQ_DENSE_MXF4=0)        */
#define VXQ_DENSE_KIND_I8X3 3    /* SBM, uniform |J|: exact int8 digit planes, kind::i8     */
#define VXQ_DENSE_KIND_F16X2 4   /* SBM, uniform |J|: two fp16 q planes (VXQ_SBM_PLANES=2)  */
#define VXQ_DENSE_KIND_BF16X3 5  /* SBM, uniform |J|: three bf16 q planes (VXQ_SBM_PLANES=3) */
#define VXQ_DENSE_KIND_J16X2 6   /* PA, general J: two fp16 J planes                        */
#define VXQ_DENSE_KIND_JQ16 7    /* SBM, general J: two fp16 J x two fp16 q planes          */

/* Build a device problem from the reference's canonical arrays:
 * rows/cols int64 with rows[k] < cols[k], sorted unique (model.py:81-104),
 * values/h fp64, offset. device = CUDA ordinal. Host pointers.
 * Dense models: rows = cols = NULL with num_couplings = n (n - 1) / 2 means the full
 * upper triangle in canonical (row-major) order -- the only canonical set of that size --
 * and only the values cross PCIe (the indices are generated on the device). */
VXQ_API int vxq_problem_create(int64_t n, int64_t num_couplings, const int64_t* rows,
                       const int64_t* cols, const double* values, const double* h,
                       double offset, int device, vxq_problem** out);
VXQ_API int vxq_problem_destroy(vxq_problem* p);
/* Generate an instance directly on the device (no host arrays).
 * family 0 = "qubo_deg6": random QUBO with mean degree ~6 -- a random graph: for each
 * variable i and c in {0,1,2} an independent Philox draw picks a partner j != i uniformly
 * (duplicates merged), Q ~ U[-1,1), converted like qubo_to_ising
 * (transforms.py:36-56) -- BASELINE config 5 at n = 2e8.  Definition: csrc/generate.cu. */
VXQ_API int vxq_problem_generate(int32_t family, int64_t n, uint64_t seed, int device,
                                 vxq_problem** out);
/* Copy the canonical model back (host or device pointers, any may be NULL): couplings
 * rows/cols/values [num_couplings] (i<j, sorted), h [n], offset. */
VXQ_API int vxq_problem_export(const vxq_problem* p, int64_t* rows, int64_t* cols,
                               double* values, double* h, double* offset);
/* info: [n, num_couplings, nnz_sym, max_row_nnz, uniform_magnitude] */
VXQ_API int vxq_problem_info(const vxq_problem* p, int64_t* info5);
/* *out = 1 if VXQ_PATH_AUTO would run an fp32 solve of `replicas` replicas on the tensor-core
 * path (solver 0 = PA, 1 = SBM; q_cap / init_noise matter for SBM on general J only).
 * Replica shards use it to choose the path once from the GLOBAL replica count, so every
 * shard computes exactly the rows the single-GPU solve would. */
VXQ_API int vxq_dense_eligible(const vxq_problem* p, int32_t solver, int64_t replicas,
                               double q_cap, double init_noise, int32_t* out);

VXQ_API int vxq_problem_lambda0(vxq_problem* p, double* out); /* max(field_scale, 1e-12) */
VXQ_API int vxq_problem_c0(vxq_problem* p, double* out);      /* 1/lambda_max(-A) or 1.0 */
/* How the automatic c0 was obtained (computes it if needed), eig_extreme(-A, "max")
 * (solvers/eigen.py:35-56): info6 = [lambda_max returned, largest Ritz value theta,
 * explicit residual ||B y - theta y|| / ||y||, Lanczos steps, method, c0]; method 0 = n <= 512
 * exact (full-dimension Lanczos with full reorthogonalisation, as eigvalsh), 1 = Lanczos to
 * ARPACK's tol 1e-8 and theta + residual, 2 = no convergence: Gershgorin bound.  Entries
 * 0-4 are NaN / -1 for a coupling-free problem (c0 = 1). */
VXQ_API int vxq_problem_eig_info(vxq_problem* p, double* info6);

VXQ_API int vxq_pa_solve(vxq_problem* p, const vxq_pa_params* prm, const vxq_run_opts* opts,
                 vxq_outputs* out);
VXQ_API int vxq_sbm_solve(vxq_problem* p, const vxq_sbm_params* prm, const vxq_run_opts* opts,
                  vxq_outputs* out);

/* Simulated annealing (annealing.py:24-74): R independent replicas, single-spin-flip
 * Metropolis sweeps in fixed index order, each replica reports the best state seen
 * (checked after every sweep).  Fields F = S A + h are kept per replica and updated in
 * O(degree) per accepted flip.  Replica r draws from Philox(seed).jumped(r): spins from
 * integers(0, 2, n), then one uniform per (sweep, spin).  energy_trace must be NULL;
 * x/m must be NULL.  Path: RESIDENT keeps each warp's fields in shared memory (small n),
 * SPARSE keeps them in HBM/L2 ([n][R] replica-contiguous). */
VXQ_API int vxq_sa_solve(vxq_problem* p, const vxq_sa_params* prm, const vxq_run_opts* opts,
                         vxq_outputs* out);

/* integrate(B, g, Q, P, ...): B given as CSR of B^T (row i lists B[j,i]),
 * Q/P [R][n] fp64 host arrays updated in place; a_sched[T] host fp64. */
VXQ_API int vxq_sbm_integrate(int64_t n, const int64_t* bt_indptr, const int32_t* bt_indices,
                      const double* bt_data, const double* g, int64_t R, double* Q,
                      double* P, const double* a_sched, int64_t T, double dt, double a0,
                      double c0, double q_cap, const vxq_run_opts* opts);

/* ---- Row-partitioned solves (multi-GPU): one session per rank ----
 * The rank updates rows [row_begin, row_end) of every replica each step; every row's state
 * is read from an exchange buffer (caller-owned device memory, rows_alloc x row_bytes,
 * globally row-indexed: PA = sign bits, SBM = q) that the caller all-gathers between steps
 * (e.g. NCCL all_gather over NVLink).  Buffer k & 1 holds state k: create() writes the
 * local rows of state 0; step(t) reads buffer t & 1 and writes the local rows of buffer
 * (t+1) & 1 on opts->stream; steps run in order.  finish() needs the buffer of the last
 * state complete on every row and returns states/energies of all replicas after the steps
 * taken (normally all T; after k < T steps: a snapshot of the T-step schedule, e.g. for
 * short-horizon trajectory checks).  x/m outputs (PA X/M, SBM Q/P) only from a session
 * over all rows [0, n).
 * solver: 0 = PA (pa params), 1 = SBM (sbm params).                                  */
typedef struct vxq_session vxq_session;
VXQ_API int vxq_exchange_row_bytes(int32_t solver, int64_t replicas, int32_t precision,
                                   int64_t* out);
VXQ_API int vxq_session_create(vxq_problem* p, int32_t solver, const vxq_pa_params* pa,
                               const vxq_sbm_params* sbm, int64_t row_begin, int64_t row_end,
                               int64_t rows_alloc, void* xbuf0, void* xbuf1,
                               const vxq_run_opts* opts, vxq_session** out);
VXQ_API int vxq_session_step(vxq_session* s, int64_t t);
VXQ_API int vxq_session_finish(vxq_session* s, vxq_outputs* out);
VXQ_API int vxq_session_destroy(vxq_session* s);

/* ---- Fused exchange over NVLink peer memory (replaces the caller's all-gather) ----
 * Every rank allocates its two exchange buffers and a flag array of `world` uint64 with
 * vxq_exchange_alloc (zeroed, IPC-shareable), shares vxq_ipc_handle() of each with the
 * other ranks (e.g. torch.distributed.all_gather_object) and opens the peers' handles with
 * vxq_ipc_open.  vxq_session_set_peers(s, world, rank, xbuf0[world], xbuf1[world],
 * flags[world]) (own pointers at [rank]) pushes state 0 of the local rows to every peer;
 * from then on vxq_session_step stores each produced word / q vector directly into every
 * rank's buffer from the step kernel, publishes "state t+1 complete" into every rank's
 * flags[rank] (release, system scope) and, before step t, waits on its own flags for
 * state t from all sources (acquire; bounded at 30 s -> VXQ_ERR_CUDA at finish).
 * Flag values are (epoch << 32) + state + 1: reuse one exchange for several sessions with
 * a larger epoch each time (same on every rank) and a barrier between sessions.
 * No caller collective is needed between steps.                                        */
#define VXQ_IPC_HANDLE_BYTES 64
VXQ_API int vxq_exchange_alloc(int device, int64_t bytes, void** out);
VXQ_API int vxq_exchange_free(void* ptr);
VXQ_API int vxq_ipc_handle(const void* dev_ptr, void* handle_out);
VXQ_API int vxq_ipc_open(const void* handle, int device, void** dev_ptr);
VXQ_API int vxq_ipc_close(void* dev_ptr);
VXQ_API int vxq_session_set_peers(vxq_session* s, int32_t world, int32_t rank,
                                  uint32_t epoch, void* const* xbuf0, void* const* xbuf1,
                                  uint64_t* const* flags);

/* Exact energies of R spin states [R][n] int8 (host, or device if
 * opts->outputs_on_device) -> energies[R] (same residency). */
VXQ_API int vxq_energies(vxq_problem* p, const int8_t* states, int64_t R, double* energies,
                 const vxq_run_opts* opts);

/* Host-only helpers (no GPU needed): the step schedules the loops use,
 * bit-exact with the reference's Python expressions.
 *   PA : lam_t = lambda0 * (1.0 - t / T)        parallel_annealing.py:42
 *   SBM: a_t   = numpy.linspace(0.0, a0, T)[t]  bifurcation.py:63          */
VXQ_API int vxq_pa_schedule(double lambda0, int64_t T, double* out);
VXQ_API int vxq_sbm_schedule(double a0, int64_t T, double* out);
/*   SA : temps[k] = T_init * pow(pow(T_final / T_init, 1 / (sweeps - 1)), k)
 *        (annealing.py:31-35; numpy may differ by an ulp -- pass params.temps for parity) */
VXQ_API int vxq_sa_schedule(double T_init, double T_final, int64_t sweeps, double* out);

VXQ_API const char* vxq_last_error(void);
VXQ_API int vxq_abi_version(void);
VXQ_API int vxq_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* VXQ_H_ */
