/*
 * airsched.h -- C ABI of the B200-native move-evaluation and selection engine
 * for arXiv 2002.11710 ("air-EMS fleet scheduling": neighbourhood search and
 * tabu search over mission-to-vehicle routes).
 *
 * Citations: "P:n" = line n of the paper's text (/root/reference/PAPER.md,
 * not needed at run time); "reading #k" = DESIGN.md's ambiguity ledger.
 *
 * Conventions (all entry points):
 *  - Every call returns as_status; outputs are written only on AS_OK.  No C++
 *    exception crosses the ABI.  as_last_error() returns a thread-local message
 *    for the last non-OK status of the calling thread.
 *  - Inputs are copied; the caller keeps its buffers.  Handles are destroyed
 *    explicitly by the caller.
 *  - Array arguments marked "(host or device)" may point to host memory or to
 *    device memory of the context's device (for example a torch CUDA tensor's
 *    data_ptr()); the library classifies them with cudaPointerGetAttributes.
 *    Host outputs are complete when the call returns; a call whose array
 *    outputs are all device pointers only enqueues work on the context's
 *    stream (callers synchronise the stream themselves).
 *  - Schedules cross the boundary in CSR form: route_ptr[V+1] (route_ptr[0] =
 *    0, non-decreasing) and route_missions[route_ptr[V]], vehicle v flying
 *    route_missions[route_ptr[v] .. route_ptr[v+1]) in order, base -> missions
 *    -> the same base (Alg. 1 line 5 "Solution" matrix).
 *  - Integer seconds everywhere; objective values are int64 seconds.
 */
#ifndef AIRSCHED_H
#define AIRSCHED_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AS_OK = 0,
    AS_ERR_INVALID_ARG = 1,      /* bad sizes, indices, ranges, null pointers */
    AS_ERR_INFEASIBLE_START = 2, /* start schedule violates con6-con9 */
    AS_ERR_INIT_FAILED = 3,      /* Alg. 1 found no schedule (O13) */
    AS_ERR_DEVICE = 4,           /* CUDA error (message in as_last_error) */
    AS_ERR_OOM = 5,              /* device allocation failed */
    AS_ERR_COMM = 6,             /* NCCL error */
    AS_ERR_UNSUPPORTED = 7       /* size outside what this build's kernels handle */
} as_status;

typedef struct as_instance as_instance; /* immutable after create; thread-safe */
typedef struct as_ctx as_ctx;           /* one device + one CUDA stream; single-threaded */
typedef struct as_comm as_comm;         /* NCCL communicator (multi-GPU); may be NULL */

/* ---------------------------------------------------------------- instance --
 * The paper's problem statement (§3): bases with a vehicle class
 * and location, missions <pickup, delivery, rho> with a
 * deadline w_n, the flight limit p and the 24 h return limit
 * (P:148).  Travel times are an input matrix of integer seconds per class
 * (the paper's d built from Eq. e1; BASELINE north_star).  Several
 * vehicles may share a base (reading #12).  All arrays are host memory and
 * are copied.
 */
typedef struct {
    int32_t n_locations;            /* NL >= 1: facilities and base sites */
    int32_t n_classes;              /* NC in [1, 4]: matrix layers l (paper: 2) */
    const int32_t *travel_s;        /* [NC][NL][NL] row-major, 0 <= T < 2^26, T[c][a][a] == 0 */
    const uint8_t *class_is_heli;   /* [NC] 1 = helicopter class (may serve rho=1 missions, con9) */
    int32_t n_bases;                /* >= 1 */
    const int32_t *base_location;   /* [n_bases] in [0, NL) */
    int32_t n_vehicles;             /* V >= 1 */
    const int32_t *vehicle_base;    /* [V] in [0, n_bases) */
    const int32_t *vehicle_class;   /* [V] in [0, NC)  (l = b_k) */
    int32_t n_missions;             /* n >= 0 */
    const int32_t *pickup_loc;      /* [n] in [0, NL) */
    const int32_t *delivery_loc;    /* [n] in [0, NL) */
    const int32_t *deadline_s;      /* [n] w_n in [1, day_length_s] */
    const uint8_t *heli_only;       /* [n] rho: 1 = helicopter required */
    int32_t flight_limit_s;         /* p > 0 (36000 = 10 h) */
    int32_t day_length_s;           /* in [flight_limit_s, 2^30) (86400) */
    int32_t no_wait;                /* 0: the paper's model -- a vehicle departs mission n at
                                     *    exactly w_n (readings #2-#6);
                                     * 1: no-wait variant (reading #40) -- it
                                     *    departs on arrival, deadlines bound arrivals.  The
                                     *    variant runs on the per-CTA kernel only: the sweep mode
                                     *    and the sharded path return AS_ERR_UNSUPPORTED. */
} as_instance_desc;

/* Validates and copies desc (AS_ERR_INVALID_ARG names the violated rule).
 * Limits: n + V < 2^20, the move-space size n(n+V)+n^2 < 2^32 - 1. */
as_status as_instance_create(const as_instance_desc *desc, as_instance **out);
void as_instance_destroy(as_instance *inst);

/* Canonical move space (O5): relocate block
 * idx = m*(n+V) + t (remove mission m, insert it before mission t, or at the
 * end of route t-n for t >= n), then swap block idx = n(n+V) + m1*n + m2. */
int64_t as_move_space_size(const as_instance *inst);
/* Valid indices per iteration for a complete schedule with every move kind
 * enabled: n(n+V-2) + n(n-1)/2 (state-independent). */
int64_t as_valid_moves_per_iter(const as_instance *inst);

/* Host-side check of a complete or partial CSR schedule against the model
 * (Eq. obj_s, con1-con9).  feasible: 1 iff complete and feasible.  objective:
 * total flight seconds (Eq. obj_s).  Pointers: host. */
as_status as_schedule_check(const as_instance *inst, const int32_t *route_ptr, const int32_t *route_missions,
                            int32_t *feasible, int64_t *objective);

/* An owned, validated copy of a schedule: one ordered route per vehicle
 * in CSR form.  Creation copies the arrays and applies as_schedule_check's rules (route_ptr[0] = 0 and
 * non-decreasing, mission ids in range and listed at most once; every mission listed unless allow_partial),
 * then stores the objective (Eq. obj_s) and feasibility (con6-con9).  The run calls take
 * the CSR arrays directly (as_schedule_get hands them out); the handle is the caller's, freed with
 * as_schedule_destroy.  Pointers: host. */
typedef struct as_schedule as_schedule;
as_status as_schedule_from_routes(const as_instance *inst, const int32_t *route_ptr, const int32_t *route_missions,
                                  int32_t allow_partial, as_schedule **out);
/* Any output may be NULL: route_ptr[V + 1], route_missions[n_assigned] (n_assigned = route_ptr[V]),
 * objective (seconds), feasible (1 iff complete and feasible), n_assigned. */
as_status as_schedule_get(const as_schedule *s, int32_t *route_ptr, int32_t *route_missions, int64_t *objective,
                          int32_t *feasible, int32_t *n_assigned);
void as_schedule_destroy(as_schedule *s);

/* ----------------------------------------------------------------- context --
 * device: CUDA ordinal.  cuda_stream: a cudaStream_t (e.g. torch's current
 * stream); NULL = the legacy default stream. */
as_status as_ctx_create(int32_t device, void *cuda_stream, as_ctx **out);
as_status as_ctx_set_stream(as_ctx *ctx, void *cuda_stream);

/* Explicit per-context overrides of the kernel choice and launch shape.  The
 * library picks every kernel and shape itself; these options exist so that the
 * test suite can force each code path (and its fallbacks) onto small inputs.
 * Nothing else changes them -- no environment variable is read.  value
 * INT64_MIN restores the automatic choice; other values must lie in
 * [-1, 2^40]; an unknown option returns AS_ERR_INVALID_ARG.  Results never
 * depend on these options (the parity tests run every path). */
enum {
    AS_OPT_SMEM_LIMIT = 0,     /* cap on dynamic shared memory per CTA, bytes */
    AS_OPT_T_SMEM,             /* 0: per-run kernel keeps the table in global memory */
    AS_OPT_WINDOW,             /* 0: batched kernel without the window scorers */
    AS_OPT_BATCH_KERNEL,       /* 1: single runs on the batched kernel; 0: never */
    AS_OPT_GRID,               /* 1: single runs on the whole-GPU kernel; 0: never */
    AS_OPT_GRID_MIN,           /* move count from which single runs use the whole-GPU kernel */
    AS_OPT_ONE_CTA,            /* 0: no one-CTA whole-GPU kernel for small single runs */
    AS_OPT_GRID_T_GLOBAL,      /* 1: whole-GPU kernel reads the table from global memory */
    AS_OPT_GRID_E_GLOBAL,      /* 1: whole-GPU kernel keeps the tabu matrix in global memory */
    AS_OPT_GRID_BLOCKS,        /* CTAs of the whole-GPU kernel */
    AS_OPT_GRID_G,             /* rows per tile of the whole-GPU kernel */
    AS_OPT_VERBOSE,            /* 1: print the dispatch decision to stderr */
    AS_OPT_RPC,                /* runs per CTA of the batched kernel */
    AS_OPT_THREADS,            /* threads per CTA of the per-run kernel */
    AS_OPT_SHARDED,            /* 1: single runs on the sharded (global-state) kernels without a comm */
    AS_OPT_GREEDY_GLOBAL,      /* 1: device Alg. 1 keeps its state in global memory */
    AS_OPT_SHARD_FUSED,        /* 0: sharded runs with a comm use the NCCL-graph path, not the fused kernel */
    AS_OPT_SHARD_FUSED_1,      /* 1: the fused kernel also with a one-rank comm */
    AS_OPT_SHARD_EMULATE,      /* sharded kernels without a comm: emulate this many ranks' slices */
    AS_OPT_SHARD_K,            /* iterations per CUDA graph of the NCCL-graph path */
    AS_OPT_XR_TIMEOUT_MS,      /* fused sharded exchange: bound on the wait for a peer (default 30000) */
    AS_OPT_PHASE_TIMES,        /* 1: the whole-GPU kernel records its per-iteration phase latencies */
    AS_OPT_NODE_COSTS,         /* 0: no global node-cost table for the global-table scorers (set before upload) */
    AS_OPT_GRID_COMPACT,       /* 0: the whole-GPU kernel keeps the empty swap tiles in its tile list */
    AS_OPT_GRID_SWAP_REC,      /* 0: no per-warp swap-row records in the whole-GPU kernel's global-table scorers */
    AS_OPT_GRID_WARPS,         /* warps per CTA of the whole-GPU kernel (1..20; default 20, 8 as one cluster) */
    AS_OPT_GRID_CLUSTER,       /* whole-GPU kernel as ONE thread-block cluster of this many CTAs (2..16; 0: never;
                                  automatic: 16 for small instances with shared-memory tables) */
    AS_OPT_COUNT
};
as_status as_ctx_set_option(as_ctx *ctx, int32_t option, int64_t value);
/* Per-iteration device latency of the last whole-GPU (k_grid) run made with AS_OPT_PHASE_TIMES = 1,
 * measured by CTA 0 with %globaltimer and summed over the iterations: out[0] its own tiles' scoring,
 * out[1] waiting for the CTA's other warps, out[2] CTA reduction + grid barrier (+ rank exchange),
 * out[3] apply, in ns; out[4] = iterations; out[5] the part of out[3] spent reading the winning key
 * from L2 after the barrier; out[6..9] lane 0's split, relink, totals + bookkeeping, and the warp's record
 * refresh inside the apply.  out holds 10 entries.  Synchronises the context's stream.
 * AS_ERR_INVALID_ARG if no such run was made. */
as_status as_ctx_grid_phases(as_ctx *ctx, int64_t *out);
/* Per CTA of that run (at most 256): tile_ns[c] = the sum over iterations of CTA c's own tile phase (loop
 * top to all of its warps done), smid[c] = the SM it ran on; *n_ctas = the CTA count.  Host buffers of 256. */
as_status as_ctx_grid_cta_phases(as_ctx *ctx, int64_t *tile_ns, int32_t *smid, int32_t *n_ctas);
void as_ctx_destroy(as_ctx *ctx);
/* Upload (and cache on ctx) the instance's device copy.  Optional: every call
 * below uploads on first use; call this to keep the upload out of a timed
 * region. */
as_status as_instance_upload(as_ctx *ctx, const as_instance *inst);

/* ------------------------------------------------------- Algorithm 1 (O13) --
 * Greedy initialisation: helicopter-only missions first, each
 * phase by ascending (deadline, id); the vehicle with the smallest cost
 * increase wins (ties: lower id); insert_mode 0 = TAIL (route end, reading
 * #23), 1 = SORTED (deadline-sorted slot).  When no vehicle fits, one
 * neighbourhood-search iteration runs on the device over the assigned missions
 * and the mission is retried once (reading #22).  Runs on the
 * device (one warp scans the vehicles per mission, a packed (increase, vehicle)
 * minimum replaces the paper's mutex-protected CurrentMin).
 * Outputs (host or device): route_ptr_out[V+1], route_missions_out[n].
 * AS_ERR_INIT_FAILED: a mission fits no vehicle with nothing assigned yet
 * (P:166), the repair found no improving move, the retry failed, or more than
 * max_repairs repairs were needed. */
as_status as_init_greedy(as_ctx *ctx, const as_instance *inst, int32_t insert_mode, int32_t max_repairs,
                         int32_t *route_ptr_out, int32_t *route_missions_out, int32_t *n_repairs_out);

/* Batched randomized starts (reading #41): Algorithm 1
 * for n_starts starts in one launch, one warp per start.  seeds[r] == 0 keeps
 * the paper's placement order; seeds[r] != 0 permutes each phase's order
 * (SplitMix64 Fisher-Yates from the top, helicopter-only phase first).  seeds:
 * [n_starts] host or device, or NULL (all 0).  Outputs, host or device:
 * route_ptr_out[n_starts][V+1], route_missions_out[n_starts][n],
 * status_out[n_starts] (AS_OK or AS_ERR_INIT_FAILED; a failed start has empty
 * routes) and n_repairs_out[n_starts], both nullable.  The outputs feed
 * as_batch_run with shared_start = 0 directly (device pointers stay on the
 * device). */
as_status as_init_greedy_batch(as_ctx *ctx, const as_instance *inst, int32_t n_starts, int32_t insert_mode,
                               int32_t max_repairs, const uint64_t *seeds, int32_t *route_ptr_out,
                               int32_t *route_missions_out, int32_t *status_out, int32_t *n_repairs_out);

/* ----------------------------------------------------------- evaluation --- */
enum { AS_MODE_NS = 0, AS_MODE_TABU = 1 };
enum { AS_FLAG_VALID = 1, AS_FLAG_FEASIBLE = 2, AS_FLAG_TABU = 4, AS_FLAG_ADMISSIBLE = 8,
       AS_FLAG_BYDEFAULT = 16 };
enum { AS_MOVE_INTER_RELOCATE = 1, AS_MOVE_INTRA_RELOCATE = 2, AS_MOVE_INTER_SWAP = 4,
       AS_MOVE_INTRA_SWAP = 8, AS_MOVE_ALL = 15 };

/* Selection key of a move (O9): (class << 63) | ((delta + 2^30) << 32) | idx,
 * class 0 = admissible, 1 = feasible but not admissible (by-default);
 * AS_KEY_NONE = invalid or infeasible.  The minimum key is the selected move:
 * smallest delta, ties to the lowest index (reading #26). */
#define AS_KEY_NONE 0xFFFFFFFFFFFFFFFFull

/* Score every canonical index of one schedule: delta (Eq. obj_s difference,
 * defined for every valid index), FEASIBLE (con6-con9 of the moved schedule),
 * TABU (some (mission, vehicle) the move places into has tabu_expiry >= iter),
 * ADMISSIBLE (TS: feasible and (not tabu or cur+delta < best_obj);
 * NS: feasible and delta < 0), BYDEFAULT (feasible, not admissible).
 * Invalid indices get delta 0, flags 0.  The schedule (host) must be feasible
 * (AS_ERR_INFEASIBLE_START otherwise); it may be partial (unlisted missions
 * are unassigned; every move touching them is invalid).
 * tabu_expiry: [n][V] int32 (host or device) or NULL (nothing tabu).
 * delta_out [N] int32, flags_out [N] uint8 (host or device, nullable),
 * best_key_out (host, nullable).  N = as_move_space_size. */
as_status as_eval_moves(as_ctx *ctx, const as_instance *inst, const int32_t *route_ptr,
                        const int32_t *route_missions, int32_t mode, const int32_t *tabu_expiry, int32_t iter,
                        int64_t best_obj, uint32_t move_mask, int32_t *delta_out, uint8_t *flags_out,
                        uint64_t *best_key_out);

/* --------------------------------------------------------------- search --- */
typedef struct {
    int32_t mode;             /* AS_MODE_NS (Alg. 2) or AS_MODE_TABU (Alg. 3) */
    int32_t tenure;           /* TabuCounter: a move applied at it is tabu during it+1..it+tenure */
    int32_t max_iters;        /* iterations (one iteration = full neighbourhood + one applied move) */
    int32_t kick;             /* relocates of the seeded kick (O12); used when seed != 0 */
    uint32_t move_mask;       /* AS_MOVE_* bits; AS_MOVE_INTER_RELOCATE alone = the paper's move set */
    int32_t strict_tabu_stop; /* TS: stop (reason 2) instead of the by-default move */
    int32_t trace_level;      /* 0 none, 1 per-iteration records, 2 + tabu-list digest */
    uint64_t seed;            /* run seed; 0 = start unchanged */
    int32_t sweep;            /* 0: north_star's global-best iteration (every move, one best per
                                 iteration).  1: the paper-literal sweep of Alg. 2 / Alg. 3 (P:294-336,
                                 P:362-415): for each vehicle i, for each mission j of route i,
                                 apply the best admissible inter-route relocate of j; one iteration =
                                 one (i, j) step, max_iters = steps; seed != 0 permutes the vehicle and
                                 mission order each sweep; kick and move_mask are ignored.
                                 Runs on the batched kernel (as_batch_run, as_tabu_run, as_nbhd_run). */
    int32_t reserved;
} as_run_params;

enum { AS_STOP_MAX_ITERS = 0, AS_STOP_LOCAL_OPT = 1, AS_STOP_NO_MOVE = 2, AS_STOP_INFEASIBLE_START = 3,
       AS_STOP_COMM_ABORT = 4   /* fused sharded run: a peer's key did not arrive within the exchange
                                   timeout; the call returns AS_ERR_COMM (the result is partial) */ };

typedef struct {
    int64_t best_obj, final_obj, start_obj;
    int32_t best_iter;        /* -1 if the start was never improved */
    int32_t iters_done, stop_reason, kicks_applied;
} as_run_result;              /* 40 bytes */

typedef struct {
    int64_t cur, best;        /* objective after the move; best so far */
    uint32_t idx;             /* applied canonical move index */
    int32_t delta;
    int32_t cls;              /* 0 admissible, 1 by-default */
    int32_t it;
} as_trace_rec;               /* 32 bytes */

/* One NS/TS run (O10/O11) from a complete feasible start (host).  Outputs:
 * result (host), best schedule CSR (host or device, nullable), trace
 * [max_iters] (host or device, nullable, trace_level >= 1), digest [max_iters]
 * FNV-1a-64 of the tabu list after each iteration (trace_level 2), tabu_out
 * [n][V] final expiry matrix (nullable).  comm: NULL = one GPU. */
as_status as_tabu_run(as_ctx *ctx, as_comm *comm, const as_instance *inst, const int32_t *start_ptr,
                      const int32_t *start_missions, const as_run_params *params, as_run_result *result,
                      int32_t *best_ptr_out, int32_t *best_missions_out, as_trace_rec *trace_out,
                      uint64_t *digest_out, int32_t *tabu_out);
/* as_tabu_run with params->mode forced to AS_MODE_NS (Alg. 2). */
as_status as_nbhd_run(as_ctx *ctx, as_comm *comm, const as_instance *inst, const int32_t *start_ptr,
                      const int32_t *start_missions, const as_run_params *params, as_run_result *result,
                      int32_t *best_ptr_out, int32_t *best_missions_out, as_trace_rec *trace_out);

/* n_runs independent runs of one instance (multi-start), one after its own
 * seeded kick (seeds[r]; params->seed is ignored).  Starts (host or device):
 * start_ptr [n_runs][V+1], start_missions [n_runs][n], or a single shared
 * start when shared_start != 0.  Outputs (host or device, nullable):
 * results [n_runs], best_ptr_out [n_runs][V+1], best_missions_out
 * [n_runs][n], trace_out [n_runs][max_iters] (trace_level >= 1).
 * best_run_out (host, nullable): run with the smallest (best_obj, run) over
 * all ranks of comm.  A run whose start is infeasible reports stop_reason
 * AS_STOP_INFEASIBLE_START; the call still succeeds.  The best-run reduction
 * packs (best_obj << 32 | global run): AS_ERR_UNSUPPORTED when V x
 * flight_limit_s >= 2^31, AS_ERR_INVALID_ARG when nranks x n_runs >= 2^32. */
as_status as_batch_run(as_ctx *ctx, as_comm *comm, const as_instance *inst, int32_t n_runs,
                       const int32_t *start_ptr, const int32_t *start_missions, int32_t shared_start,
                       const as_run_params *params, const uint64_t *seeds, as_run_result *results,
                       int32_t *best_ptr_out, int32_t *best_missions_out, as_trace_rec *trace_out,
                       int64_t *best_run_out);

/* Several instances in one launch ("independent multi-start runs or instances",
 * BASELINE north_star): job j runs jobs[j].n_runs independent runs of
 * jobs[j].inst from jobs[j]'s start (host or device CSR), all with *params; the
 * runs are numbered job after job (run = sum of the earlier jobs' n_runs + r)
 * and seeds / results / trace are indexed by that number.  Each CTA of the
 * batched kernel stages the instance of the job it serves, so many small
 * instances fill the GPU together.  Every instance must fit the compact layout
 * (NL and n+V < 65536, <= 2 classes, waiting model), else AS_ERR_UNSUPPORTED.
 * best_ptr_out / best_missions_out (nullable): the runs' best schedules packed
 * job after job ([n_runs][V_j+1] and [n_runs][n_j] per job).  best_run_out: the
 * run with the smallest (best objective, run number), over every rank with a
 * communicator (run numbers then offset by rank x total runs). */
typedef struct {
    const as_instance *inst;
    const int32_t *start_ptr;       /* [V+1] */
    const int32_t *start_missions;  /* [n] */
    int32_t n_runs;                 /* >= 1 */
    int32_t reserved;               /* 0 */
} as_job;

as_status as_batch_run_jobs(as_ctx *ctx, as_comm *comm, int32_t n_jobs, const as_job *jobs,
                            const as_run_params *params, const uint64_t *seeds, as_run_result *results,
                            int32_t *best_ptr_out, int32_t *best_missions_out, as_trace_rec *trace_out,
                            int64_t *best_run_out);

/* ------------------------------------------------------------- multi-GPU --
 * One process per GPU.  Rank 0 creates a 128-byte NCCL unique id, the caller
 * shares it (e.g. through torch.distributed), every rank calls as_comm_init on
 * its own context.  With a communicator, as_tabu_run / as_nbhd_run shard the
 * move space of ONE instance across the ranks (every rank must pass the same
 * instance, start and params): each iteration every rank scores its slice,
 * an 8-byte ncclAllReduce(MIN) selects the global best packed key, and every
 * rank applies it to its replica -- the trace is identical to one GPU.
 * as_batch_run with a communicator runs each rank's own runs and then reduces
 * the best (objective, global run) over all ranks (best_run_out). */
as_status as_comm_unique_id(void *uid_out /* 128 bytes, host */);
as_status as_comm_init(as_ctx *ctx, int32_t nranks, int32_t rank, const void *uid /* 128 bytes, host */,
                       as_comm **out);
void as_comm_destroy(as_comm *comm);
/* After as_batch_run (with or without a communicator): the best run over all
 * ranks -- the minimum of (best_obj << 32 | global run), global run = rank *
 * n_runs + r (every rank runs n_runs runs); as_batch_run already reduced it on
 * the device with ncclAllReduce(MIN).  If ptr_out/ms_out are given, the owner
 * rank broadcasts that run's best schedule (CSR) to every rank (ncclBroadcast);
 * run_best_ptr/run_best_ms are this rank's per-run best schedules as written
 * by as_batch_run ([n_runs][V+1], [n_runs][n], host or device).  Outputs host. */
as_status as_batch_gather_best(as_ctx *ctx, as_comm *comm, int32_t n_runs, const int32_t *run_best_ptr,
                               const int32_t *run_best_ms, int64_t *best_run_out, int64_t *best_obj_out,
                               int32_t *ptr_out, int32_t *ms_out);

/* The contiguous tile range [tile_lo, tile_hi) of the flat neighbourhood tile
 * list that `rank` scores in a sharded run on GPUs with n_sm SMs (host logic;
 * the split balances scored moves).  weight_*: moves in the rank's range and
 * in total.  Pointers: host, nullable. */
as_status as_shard_plan(const as_instance *inst, int32_t nranks, int32_t rank, int32_t n_sm, int32_t *tile_lo,
                        int32_t *tile_hi, int32_t *tile_total, int64_t *weight_rank, int64_t *weight_total);

/* Device time of the last search/eval call's kernels on ctx's stream (ms),
 * measured with CUDA events around the launches. */
float as_ctx_last_kernel_ms(const as_ctx *ctx);
/* Number of kernels the library launched on ctx since creation. */
int64_t as_ctx_kernel_launches(const as_ctx *ctx);

const char *as_last_error(void);
const char *as_version(void);

#ifdef __cplusplus
}
#endif
#endif
