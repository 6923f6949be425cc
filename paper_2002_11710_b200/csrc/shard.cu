// shard.cu -- one instance whose move space is SHARDED across GPUs (config C5 at
// G = 2/4/8).
//
// Every rank keeps a full replica of the (small) run state in global memory
// and owns a contiguous range of the flat tile list (score.cuh).  One
// iteration is three stream-ordered steps, captured K at a time in a CUDA graph:
//   k_shard_eval   : the rank's tiles -> one packed 64-bit key (atomicMin);
//   ncclAllReduce  : 8-byte MIN over NVLink / NVSwitch (ncclUint64);
//   k_shard_apply  : every rank applies the same winning move to its replica.
// The min of packed keys is order-independent, so the move sequence is
// identical to the single-GPU kernels for any number of ranks.
#include <cuda_runtime.h>

#include <cstdint>

#include "compact.cuh"
#include "engine.cuh"
#include "launch.h"
#include "score.cuh"

namespace airsched {

struct ShardViews {
    const void *T;      // padded table
    int4 *CS4, *RS4;
    uint8_t *MH, *CH;
    uint32_t *VC, *LK;
    int32_t *F, *E, *BS;
    ShardCtl *ctl;
    int NLp;
};

template <class TT>
__device__ __forceinline__ void shard_views(const DevInst &I, const ShardViews &SV, CompactMV<TT> &M,
                                            CompactRV<int32_t> &R) {
    M.T = reinterpret_cast<const TT *>(SV.T);
    M.CS = reinterpret_cast<const unsigned char *>(SV.CS4);
    M.MH = SV.MH; M.VC = SV.VC; M.CH = SV.CH;
    M.n = I.n; M.V = I.V; M.NL = I.NL; M.NLp = SV.NLp; M.P = I.P; M.DAY = I.DAY;
    unsigned char *RSb = reinterpret_cast<unsigned char *>(SV.RS4);
    unsigned char *LKb = reinterpret_cast<unsigned char *>(SV.LK);
    R.succ.base = LKb; R.pred.base = LKb;
    R.veh.base = RSb; R.endc.base = RSb; R.depc.base = RSb; R.inc.base = RSb; R.svco.base = RSb;
    R.pick_s.base = reinterpret_cast<unsigned char *>(SV.CS4);
    R.w_s.base = reinterpret_cast<unsigned char *>(SV.CS4);
    R.F = SV.F; R.E = SV.E;
}

// Build the replica from the start CSR, apply the seeded kick (one CTA).
template <class TT>
__global__ void k_shard_init(SearchArgs A, ShardViews SV) {
    const DevInst &I = A.inst;
    const int n = I.n, V = I.V, S = n + V, NC = I.NC;
    const int tid = threadIdx.x;
    for (int x = tid; x < S; x += blockDim.x) {
        int4 r;
        if (x < n) {
            r.x = I.w[x];
            r.y = (I.pick[x] & 0xFFFF) | (I.del[x] << 16);
            r.z = I.svc[x];
            r.w = NC > 1 ? I.svc[n + x] : 0;
        } else {
            r.x = I.DAY;
            r.y = (I.vloc[x - n] & 0xFFFF) | (I.vloc[x - n] << 16);
            r.z = 0;
            r.w = 0;
        }
        SV.CS4[x] = r;
    }
    for (int i = tid; i < n; i += blockDim.x) SV.MH[i] = I.heli[i];
    for (int i = tid; i < V; i += blockDim.x) {
        int c = I.vcls8[i];
        SV.VC[i] = (uint32_t)c | ((uint32_t)I.cls_heli[c] << 8) | ((uint32_t)I.vloc[i] << 16);
    }
    for (int i = tid; i < NC; i += blockDim.x) SV.CH[i] = I.cls_heli[i];
    if (SV.E)
        for (int i = tid; i < n * V; i += blockDim.x) SV.E[i] = -1;
    CompactMV<TT> M;
    CompactRV<int32_t> R;
    shard_views<TT>(I, SV, M, R);
    for (int x = tid; x < S; x += blockDim.x) R.veh[x] = x < n ? (int16_t)-1 : (int16_t)(x - n);
    __syncthreads();
    for (int v = tid; v < V; v += blockDim.x) {
        int prev = n + v;
        for (int i = A.start_ptr[v]; i < A.start_ptr[v + 1]; i++) {
            int m = A.start_ms[i];
            R.veh[m] = (int16_t)v;
            R.succ[prev] = (uint16_t)m;
            R.pred[m] = (uint16_t)prev;
            prev = m;
        }
        R.succ[prev] = (uint16_t)(n + v);
        R.pred[n + v] = (uint16_t)prev;
    }
    __syncthreads();
    for (int x = tid; x < S; x += blockDim.x) refresh_slot(M, R, x);
    __syncthreads();
    for (int v = tid; v < V; v += blockDim.x) {
        int f = 0, x = R.succ[n + v];
        for (int g = 0; x < n && g <= n; g++) { f += R.inc[x]; x = R.succ[x]; }
        SV.F[v] = f + R.inc[n + v];
    }
    __syncthreads();
    if (tid == 0) {
        int kicks = 0;
        if (A.seed != 0 && n > 0) {
            uint64_t s = A.seed;
            const uint64_t Rb = (uint64_t)n * (uint64_t)S;
            for (int k = 0; k < A.kick; k++)
                for (int tr = 0; tr < 64; tr++) {
                    uint32_t idx = (uint32_t)(splitmix64_next(s) % Rb);
                    MoveEval e = eval_index(M, R, idx, 0xFu, 0);
                    if (e.valid && e.feasible) {
                        apply_move(M, R, idx, e, 0, 0, false);
                        kicks++;
                        break;
                    }
                }
        }
        long long c = 0;
        for (int v = 0; v < V; v++) c += SV.F[v];
        ShardCtl *ctl = SV.ctl;
        ctl->cur = ctl->best = ctl->start = c;
        ctl->it = 0;
        ctl->best_it = -1;
        ctl->stop = 0;
        ctl->kicks = kicks;
        ctl->key = KEY_NONE;
    }
    __syncthreads();
    for (int x = tid; x < S; x += blockDim.x) SV.BS[x] = (int32_t)(SV.LK[x] & 0xFFFF);
}

// Score this rank's tiles [tlo, thi) of the current state.
template <bool TABU, class TT, bool FULL>
__global__ void __launch_bounds__(768, 1) k_shard_eval(SearchArgs A, ShardViews SV, int G, int tlo, int thi) {
    const ShardCtl *ctl = SV.ctl;
    if (ctl->stop) return;
    const DevInst &I = A.inst;
    const int n = I.n, V = I.V, S = n + V;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    __shared__ unsigned long long red[32];
    CompactMV<TT> M;
    CompactRV<int32_t> R;
    shard_views<TT>(I, SV, M, R);
    ScoreCtx<TT, int32_t> SC;
    SC.Ts = reinterpret_cast<const TT *>(SV.T);
    SC.Tt = A.inst.tsym ? SC.Ts : reinterpret_cast<const TT *>(A.inst.TpadT);
    SC.TD = sizeof(TT) == 2 ? A.inst.TDg : nullptr;
    SC.RR = nullptr;
    SC.SR = nullptr;
    SC.CS4 = SV.CS4; SC.MH = SV.MH; SC.VC = SV.VC; SC.RS4 = SV.RS4;
    SC.LK = SV.LK; SC.F = SV.F; SC.E = SV.E; SC.Et = nullptr;
    SC.n = n; SC.V = V; SC.S = S; SC.NL = I.NL; SC.NLp = SV.NLp; SC.P = I.P; SC.Rb = (uint32_t)n * (uint32_t)S;
    SC.mask = A.mask;
    SC.one = A.one; SC.neg = -A.one;
    const GridTiles GT = grid_tiles(n, V, G);
    const int it = ctl->it;
    const long long cur = ctl->cur, best = ctl->best;
    uint64_t kmin = score_tiles<TABU, FULL, true>(SC, M, R, GT, tlo, thi, blockIdx.x * nwarps + warp, gridDim.x * nwarps,
                                            it, cur, best, lane);
    kmin = wmin(kmin);
    if (lane == 0) red[warp] = kmin;
    __syncthreads();
    if (warp == 0) {   // CTA minimum by one warp
        const uint64_t k = wmin(lane < nwarps ? red[lane] : KEY_NONE);
        if (lane == 0 && k != KEY_NONE) atomicMin(&SV.ctl->key, (unsigned long long)k);
    }
}

// Apply the (all-reduced) winning key to this rank's replica.
template <bool TABU, class TT>
__global__ void k_shard_apply(SearchArgs A, ShardViews SV) {
    ShardCtl *ctl = SV.ctl;
    if (ctl->stop) return;
    const DevInst &I = A.inst;
    const int S = I.n + I.V;
    CompactMV<TT> M;
    CompactRV<int32_t> R;
    shard_views<TT>(I, SV, M, R);
    __shared__ int improved;
    if (threadIdx.x == 0) {
        const uint64_t k = ctl->key;
        const int it = ctl->it;
        int stop = 0;
        improved = 0;
        if (it >= A.max_iters) stop = AS_STOP_MAX_ITERS + 100;   // guard: graph replays past max_iters
        else if (k == KEY_NONE) stop = AS_STOP_NO_MOVE;
        else if (key_cls(k) == 1 && (!TABU || A.strict_tabu_stop)) stop = TABU ? AS_STOP_NO_MOVE : AS_STOP_LOCAL_OPT;
        if (stop) {
            ctl->stop = stop;
        } else {
            const uint32_t idx = key_idx(k);
            MoveEval e = eval_index(M, R, idx, A.mask, it);
            apply_move(M, R, idx, e, it, A.tenure, TABU);
            const long long c = ctl->cur + e.delta;
            ctl->cur = c;
            if (c < ctl->best) {
                ctl->best = c;
                ctl->best_it = it;
                improved = 1;
            }
            if (A.trace) {
                as_trace_rec tr;
                tr.cur = c;
                tr.best = ctl->best;
                tr.idx = idx;
                tr.delta = e.delta;
                tr.cls = key_cls(k);
                tr.it = it;
                A.trace[it] = tr;
            }
            ctl->it = it + 1;
            if (it + 1 >= A.max_iters) ctl->stop = AS_STOP_MAX_ITERS + 100;
        }
        ctl->key = KEY_NONE;
    }
    __syncthreads();
    if (improved)
        for (int x = threadIdx.x; x < S; x += blockDim.x) SV.BS[x] = (int32_t)(SV.LK[x] & 0xFFFF);
}

__global__ void k_shard_finish(SearchArgs A, ShardViews SV) {
    if (threadIdx.x || blockIdx.x) return;
    const ShardCtl *ctl = SV.ctl;
    const int n = A.inst.n, V = A.inst.V;
    if (A.results) {
        as_run_result *res = A.results;
        res->start_obj = ctl->start;
        res->best_obj = ctl->best;
        res->final_obj = ctl->cur;
        res->best_iter = ctl->best_it;
        res->iters_done = ctl->it;
        res->stop_reason = ctl->stop >= 100 || ctl->stop == 0 ? AS_STOP_MAX_ITERS : ctl->stop;
        res->kicks_applied = ctl->kicks;
    }
    if (A.best_ptr) {
        int pos = 0;
        for (int v = 0; v < V; v++) {
            A.best_ptr[v] = pos;
            int x = SV.BS[n + v];
            for (int g = 0; x < n && g < n; g++) { A.best_ms[pos++] = x; x = SV.BS[x]; }
        }
        A.best_ptr[V] = pos;
    }
    if (A.tabu_out && SV.E)
        for (int i = 0; i < n * V; i++) A.tabu_out[i] = SV.E[i];
}

// ---- host launchers -----------------------------------------------------------
static ShardViews make_views(const ShardBufs &B, const void *Tpad, int NLp) {
    ShardViews SV;
    SV.T = Tpad; SV.CS4 = B.CS4; SV.RS4 = B.RS4; SV.MH = B.MH; SV.CH = B.CH; SV.VC = B.VC; SV.LK = B.LK;
    SV.F = B.F; SV.E = B.E; SV.BS = B.BS; SV.ctl = B.ctl; SV.NLp = NLp;
    return SV;
}

cudaError_t launch_shard_init(const SearchArgs &A, const ShardBufs &B, const void *Tpad, int tbytes, cudaStream_t st) {
    const int NLp = padded_stride(A.inst.NL, tbytes);
    ShardViews SV = make_views(B, Tpad, NLp);
    if (tbytes == 2) k_shard_init<uint16_t><<<1, 256, 0, st>>>(A, SV);
    else k_shard_init<int32_t><<<1, 256, 0, st>>>(A, SV);
    return cudaGetLastError();
}

cudaError_t launch_shard_eval(const SearchArgs &A, const ShardBufs &B, const void *Tpad, int tbytes, int mode, int G,
                              int tlo, int thi, int blocks, cudaStream_t st) {
    const int NLp = padded_stride(A.inst.NL, tbytes);
    ShardViews SV = make_views(B, Tpad, NLp);
    const bool full = (A.mask & 15u) == 15u && A.inst.svcpos;
    if (mode == 1) {
        if (tbytes == 2) {
            if (full) k_shard_eval<true, uint16_t, true><<<blocks, 768, 0, st>>>(A, SV, G, tlo, thi);
            else k_shard_eval<true, uint16_t, false><<<blocks, 768, 0, st>>>(A, SV, G, tlo, thi);
        } else {
            k_shard_eval<true, int32_t, false><<<blocks, 768, 0, st>>>(A, SV, G, tlo, thi);
        }
    } else {
        if (tbytes == 2) {
            if (full) k_shard_eval<false, uint16_t, true><<<blocks, 768, 0, st>>>(A, SV, G, tlo, thi);
            else k_shard_eval<false, uint16_t, false><<<blocks, 768, 0, st>>>(A, SV, G, tlo, thi);
        } else {
            k_shard_eval<false, int32_t, false><<<blocks, 768, 0, st>>>(A, SV, G, tlo, thi);
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_shard_apply(const SearchArgs &A, const ShardBufs &B, const void *Tpad, int tbytes, int mode,
                               cudaStream_t st) {
    const int NLp = padded_stride(A.inst.NL, tbytes);
    ShardViews SV = make_views(B, Tpad, NLp);
    if (mode == 1) {
        if (tbytes == 2) k_shard_apply<true, uint16_t><<<1, 256, 0, st>>>(A, SV);
        else k_shard_apply<true, int32_t><<<1, 256, 0, st>>>(A, SV);
    } else {
        if (tbytes == 2) k_shard_apply<false, uint16_t><<<1, 256, 0, st>>>(A, SV);
        else k_shard_apply<false, int32_t><<<1, 256, 0, st>>>(A, SV);
    }
    return cudaGetLastError();
}

cudaError_t launch_shard_finish(const SearchArgs &A, const ShardBufs &B, cudaStream_t st) {
    ShardViews SV = make_views(B, nullptr, 0);
    k_shard_finish<<<1, 1, 0, st>>>(A, SV);
    return cudaGetLastError();
}

// Best run of a batch: min over runs of (best_obj << 32 | global run).
__global__ void k_batch_best(const as_run_result *res, int n_runs, int64_t run_offset, unsigned long long *key) {
    unsigned long long k = KEY_NONE;
    for (int r = threadIdx.x; r < n_runs; r += blockDim.x) {
        if (res[r].stop_reason == AS_STOP_INFEASIBLE_START) continue;
        const unsigned long long c = ((unsigned long long)res[r].best_obj << 32) | (unsigned long long)(run_offset + r);
        k = c < k ? c : k;
    }
    __shared__ unsigned long long red[32];
    k = wmin(k);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) k = red[w] < k ? red[w] : k;
        *key = red[0] < k ? red[0] : k;
    }
}

cudaError_t launch_batch_best(const as_run_result *res, int n_runs, int64_t run_offset, unsigned long long *key,
                              cudaStream_t st) {
    k_batch_best<<<1, 256, 0, st>>>(res, n_runs, run_offset, key);
    return cudaGetLastError();
}

// Tile weights (scored moves per tile, approximately) for the rank split.
int grid_tile_count(int n, int V, int G) { return grid_tiles(n, V, G).n_total; }
int grid_tile_count_compact(int n, int V, int G) {
    const GridTiles T = grid_tiles(n, V, G);
    return T.n_reloc + compact_swap_count(n, V, G) + T.nAdj;
}

void shard_plan(int n, int V, int G, int nranks, int rank, int *tlo, int *thi, int64_t *weight_total,
                int64_t *weight_rank) {
    const GridTiles GT = grid_tiles(n, V, G);
    const int S = n + V;
    auto w = [&](int tile) -> int64_t {
        if (tile < GT.n_reloc) {
            const int c = tile % GT.nTC, g = tile / GT.nTC;
            const int rows = std::min(n, (g + 1) * G) - g * G;
            const int cols = std::min(S, (c + 1) * 32 * KR) - c * 32 * KR;
            return (int64_t)std::max(rows, 0) * cols;
        } else if (tile < GT.n_reloc + GT.n_swap) {
            const int r = tile - GT.n_reloc;
            const int j = r % GT.nSC, g = r / GT.nSC;
            const int hi = n - j * 32 * KS, lo = hi - 32 * KS;
            const int m_lo = g * G, m_hi = std::min(hi - 1, m_lo + G);
            int64_t s = 0;
            for (int m1 = m_lo; m1 < m_hi; m1++) s += hi - std::max(lo, m1 + 1);
            return s;
        }
        return 32;
    };
    std::vector<int64_t> pre(GT.n_total + 1, 0);
    for (int t = 0; t < GT.n_total; t++) pre[t + 1] = pre[t] + w(t);
    const int64_t total = pre[GT.n_total];
    auto cut = [&](int r) -> int {
        if (r <= 0) return 0;
        if (r >= nranks) return GT.n_total;
        const int64_t target = total * r / nranks;
        return (int)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
    };
    *tlo = cut(rank);
    *thi = cut(rank + 1);
    if (weight_total) *weight_total = total;
    if (weight_rank) *weight_rank = pre[*thi] - pre[*tlo];
}

}  // namespace airsched
