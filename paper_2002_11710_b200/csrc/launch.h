// launch.h -- host <-> kernel interface inside the library (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include <nccl.h>

#include "airsched.h"
#include "engine.cuh"

struct ncclDevComm;

namespace airsched {

// One run's state in global memory (dump path).
struct RunViewG {
    int32_t *succ, *pred, *veh, *endc, *depc, *inc, *svco, *pick_s, *w_s, *F, *E;
    int32_t *arr, *sl, *pos, *slp;   // no-wait variant only (f3)
};

struct SearchArgs {
    DevInst inst;
    int32_t one, neg;                      // == 1, -1 (opaque multipliers for FMA-pipe adds; set by the host)
    int32_t n_runs;
    const int32_t *start_ptr, *start_ms;   // [R][V+1], [R][n] or shared
    int32_t shared_start;
    const uint64_t *seeds;                 // [R] or null -> seed
    uint64_t seed;
    int32_t kick, tenure, max_iters, strict_tabu_stop;
    int32_t sweep;                         // f1: paper-literal (i, j) sweep (Alg. 2 / 3)
    uint32_t mask;
    int32_t T_smem, E_smem;
    int32_t *E_global;                     // [R][n][V] when !E_smem
    as_run_result *results;                // [R]
    int32_t *best_ptr, *best_ms;           // [R][V+1], [R][n]
    as_trace_rec *trace;                   // [R][max_iters]
    uint64_t *digest;                      // [R][max_iters]
    int32_t *tabu_out;                     // [R][n][V]
};

// k_grid warps per CTA (one CTA per SM): 20 leaves 96 registers per thread (no spills in the scorers);
// measured against 24 and 16 (profiles/r02/kgrid_warps_ab.jsonl): C1 +7 %, C2 +6 %, C4 +5 %, C5 +-0 vs 24;
// 16 is slower on C1 (one CTA) and C5 (throughput)
constexpr int GRID_WARPS = 20;

struct BatchLayout {
    int T, CS, MH, VC, CH, TT, TD, TDT;   // CTA-wide part (window scorers: TT transposed table when
                                          // asymmetric, TD node costs d_c(x, m) as [c][x][m] and TDT as [c][m][x])
    int shared_bytes;
    int RS, LK, BS, F, E, PM, SN;   // per-run part (offsets inside a run block); PM/SN: sweep order (f1)
    int TB, RG, WB;                 // window scorers: tabu bits, tabu-write ring, window buffer
    int NR;                         // no-wait variant: per-slot {arrival, suffix slack, position} records
    int run_bytes;
};

// One instance of a multi-instance batch (as_batch_run_jobs).
struct BatchJob {
    DevInst inst;
    const int32_t *start_ptr, *start_ms;   // the job's start schedule (device)
    BatchLayout L;
    int NLp, RPC;                           // padded table stride, runs per CTA
    int run0;                               // global index of the job's first run
    int64_t bp_off, bm_off;                 // offsets of its runs' best schedules in the packed outputs
    int64_t e_off;                          // offset of its runs' tabu matrices in SearchArgs::E_global (window scorers)
};

struct GridLayout {
    int T, CS, MH, VC, CH, RS, LK, F, E, red, RR, SP, ST, SR, NR, total;   // shared-memory byte offsets per CTA
};

struct GridArgs {
    int NLp;                       // padded row stride of the travel-time table
    GridLayout L;
    int T_smem, E_smem;            // table / tabu matrix staged in shared memory?
    int ebytes;                    // tabu expiry width: 2 when max_iters + tenure < 32767, else 4
    const void *Tglobal;           // padded table in global memory (uint16 or int32)
    int32_t *Eglobal;              // [n][V] tabu matrix when !E_smem
    int32_t *Etglobal;             // [V][n] its transpose (identical values), when !E_smem
    int32_t *BS;                   // [S] best-schedule successor array
    unsigned long long *gkey;      // [3] triple-buffered grid-wide key, KEY_NONE at launch
    int G;                         // rows per tile
    int tlo, thi;                  // this launch's slice of the flat tile list (all tiles: 0, n_total)
    int compact;                   // 1: the list without empty swap tiles (single GPU; score.cuh GridTiles::swp)
    int swap_rec;                  // 1: per-warp swap-row record scratch in shared memory (ScoreCtx::SR)
    int cluster;                   // > 1: the grid is ONE cluster of this many CTAs (k_grid<..., CL>)
    // fused sharded run (one k_grid per rank): after the grid minimum, CTA 0 stores the rank's key
    // and a tag into every peer's symmetric window slot over NVLink and waits (bounded) for the
    // peers' tags of this iteration in its own window (grid.cu rank_exchange)
    int xr, xr_nranks, xr_rank;
    unsigned xr_epoch;             // per-call run epoch (same on every rank), high half of the tags
    unsigned long long xr_timeout_ns;   // bound on the wait for the peers' keys
    ncclWindow_t xr_win;           // symmetric window: [3][nranks] {key, tag} u64 pairs
    unsigned long long *gkey2;     // [3] the all-ranks winner per slot
    unsigned long long *phase_ns;  // [5] per-phase latency sums of CTA 0 + iterations (AS_OPT_PHASE_TIMES), or null
};

// Sharded single-instance run (shard.cu): replica state in global memory.
struct ShardCtl {
    long long cur, best, start;
    int it, best_it, stop, kicks;
    unsigned long long key;     // this iteration's key (all-reduced with MIN across ranks)
};

struct ShardBufs {
    int4 *CS4, *RS4;
    uint8_t *MH, *CH;
    uint32_t *VC, *LK;
    int32_t *F, *E, *BS;
    ShardCtl *ctl;
};

cudaError_t launch_shard_init(const SearchArgs &A, const ShardBufs &B, const void *Tpad, int tbytes, cudaStream_t st);
cudaError_t launch_shard_eval(const SearchArgs &A, const ShardBufs &B, const void *Tpad, int tbytes, int mode, int G,
                              int tlo, int thi, int blocks, cudaStream_t st);
cudaError_t launch_shard_apply(const SearchArgs &A, const ShardBufs &B, const void *Tpad, int tbytes, int mode,
                               cudaStream_t st);
cudaError_t launch_shard_finish(const SearchArgs &A, const ShardBufs &B, cudaStream_t st);
cudaError_t launch_batch_best(const as_run_result *res, int n_runs, int64_t run_offset, unsigned long long *key,
                              cudaStream_t st);
void shard_plan(int n, int V, int G, int nranks, int rank, int *tlo, int *thi, int64_t *weight_total,
                int64_t *weight_rank);
int grid_tile_count(int n, int V, int G);
int grid_tile_count_compact(int n, int V, int G);

int grid_cluster_capacity(int mode, int tbytes, int ebytes, bool full, int cl, int threads, size_t smem);
size_t grid_smem_bytes(int n, int V, int NL, int NC, int tbytes, int ebytes, bool T_smem, bool E_smem, bool tabu,
                       bool swap_rec, int G, bool nw);
cudaError_t launch_grid(const SearchArgs &A, GridArgs GA, int mode, int tbytes, int blocks, int threads, size_t smem,
                        cudaStream_t st);
cudaError_t launch_pad_table(const int32_t *T, void *out, int NC, int NL, int NLp, int tbytes, bool transpose,
                             cudaStream_t st);
int padded_stride_host(int NL, int tbytes);

size_t search_smem_bytes(int n, int V, int NL, int NC, bool T_smem, bool E_smem, bool nw);
cudaError_t launch_build_state(const DevInst &I, const int32_t *ptr, const int32_t *ms, RunViewG &G, cudaStream_t st);
cudaError_t launch_eval_dump(const DevInst &I, const RunViewG &G, int mode, int it, long long cur, long long best,
                             uint32_t mask, int32_t *delta, uint8_t *flags, unsigned long long *best_key, uint64_t N,
                             int n_sm, cudaStream_t st);
cudaError_t launch_search(const SearchArgs &A, int mode, int n_runs, int threads, size_t smem, cudaStream_t st);
void batch_smem(int n, int V, int NL, int NC, int tbytes, int ebytes, bool tabu, size_t *shared_bytes,
                size_t *run_bytes, bool win = false, int tenure = 0, bool tsym = true, bool nw = false);
// win: the WINDOW scorers (window.cuh): every move kind, svcpos, uint16 table, V <= 32, tenure <= WIN_MAX_TENURE,
// not the sweep; the tabu matrix is SearchArgs::E_global ([R][n][V] int32)
constexpr int WIN_MAX_TENURE = 64;
cudaError_t launch_batch(const SearchArgs &A, int mode, int RPC, int tbytes, int ebytes, size_t smem, cudaStream_t st,
                         bool win = false);
BatchLayout batch_layout_host(int n, int V, int NL, int NC, int tbytes, int ebytes, bool tabu, bool win = false,
                              int tenure = 0, bool tsym = true);
cudaError_t launch_batch_jobs(const SearchArgs &A, const BatchJob *jobs, const int4 *cta, int n_cta, int threads,
                              size_t smem, int mode, int tbytes, int ebytes, bool full, cudaStream_t st,
                              bool win = false);
size_t greedy_smem_bytes(const DevInst &I, int warps, bool T_smem, bool state_smem);
size_t greedy_state_bytes(const DevInst &I);
cudaError_t launch_greedy(const DevInst &I, int n_starts, int insert_mode, int max_repairs, const uint64_t *seeds,
                          int32_t *order_scratch, int32_t *state_global, int warps, bool T_smem, bool state_smem,
                          int32_t *ptr_out, int32_t *ms_out, int32_t *status_out, int32_t *nrep_out, cudaStream_t st);
cudaError_t launch_build_td(const int32_t *T, const int32_t *pick, const int32_t *del, const int32_t *vloc,
                            uint16_t *TD, int n, int V, int NL, int NC, cudaStream_t st);
cudaError_t launch_svc(const int32_t *T, const int32_t *pick, const int32_t *del, int32_t *svc, int n, int NL, int NC,
                       cudaStream_t st);

}  // namespace airsched
