// greedy.cu -- Algorithm 1 on the device, one
// warp per start.
//
//   k_greedy_order : the paper's placement order, once per launch -- phase
//                    (helicopter-only missions first, lines 6-42 / 43-77), then
//                    deadline ("smallest value in MissionTimes", lines 8 / 45),
//                    then id; one thread per mission computes its rank.
//   k_greedy<NW>   : per start, lane 0 permutes each phase of that order with
//                    the start's seed (reading #41; seed 0 keeps the
//                    paper's order).  Per mission the lanes stride the vehicles
//                    (the paper's "for i <- 1 to number of bases", which its CUDA
//                    variant gave one thread per base): each lane finds
//                    its vehicle's slot (tail, or the deadline-sorted slot,
//                    P:163), checks compatibility (lines 10-12), the two links
//                    (lines 13-28) and the flight limit (lines 29-31), and the
//                    warp takes the smallest (cost increase, vehicle) by a packed
//                    64-bit min -- the paper's mutex-protected CurrentMin
//                    (lines 32-34) made deterministic.  No vehicle: one
//                    NS iteration over the assigned missions (lines 36-37,
//                    P:213; reading #22) scored by the whole warp over
//                    the canonical move space with the engine's arithmetic,
//                    then one retry.
//
// The state is the int32 RunView of engine.cuh (wide layout), per warp in shared
// memory when it fits, else in global scratch.
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.cuh"
#include "launch.h"

namespace airsched {

__global__ void k_greedy_order(DevInst I, int32_t *order) {
    const int n = I.n;
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) {
        const int pm = I.heli[m] ? 0 : 1, wm = I.w[m];
        int rank = 0;
        for (int x = 0; x < n; x++) {
            const int px = I.heli[x] ? 0 : 1, wx = I.w[x];
            rank += (px < pm) || (px == pm && (wx < wm || (wx == wm && x < m)));
        }
        order[rank] = m;
    }
}

struct GreedyArgs {
    DevInst inst;
    int n_starts, insert_mode, max_repairs, T_smem, state_smem, warps;
    const uint64_t *seeds;       // [R] or null (all 0)
    const int32_t *base_order;   // [n] from k_greedy_order
    int32_t *state_global;       // [R][words] when !state_smem
    int32_t *ptr_out, *ms_out;   // [R][V+1], [R][n]
    int32_t *status_out, *nrep_out;
};

// int32 words of one start's state
__host__ __device__ inline int greedy_state_words(int n, int V, bool nw) {
    const int S = n + V;
    return (9 + (nw ? 4 : 0)) * S + V + n + 2;
}

template <bool NW>
__global__ void k_greedy(GreedyArgs G) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const DevInst &I = G.inst;
    const int n = I.n, V = I.V, S = n + V;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int run = blockIdx.x * G.warps + warp;

    int32_t *Ts = reinterpret_cast<int32_t *>(smem_raw);
    const int nT = I.NC * I.NL * I.NL;
    if (G.T_smem)
        for (int i = threadIdx.x; i < nT; i += blockDim.x) Ts[i] = I.T[i];
    __syncthreads();
    if (run >= G.n_starts) return;

    const int words = greedy_state_words(n, V, NW);
    int32_t *st = G.state_smem ? reinterpret_cast<int32_t *>(smem_raw + (G.T_smem ? ((nT * 4 + 15) & ~15) : 0)) +
                                     (size_t)warp * words
                               : G.state_global + (size_t)run * words;
    MissionView M;
    M.T = G.T_smem ? Ts : I.T; M.del = I.del; M.heli = I.heli; M.svc = I.svc; M.vcls = I.vcls8; M.vloc = I.vloc;
    M.clsheli = I.cls_heli; M.n = n; M.V = V; M.NL = I.NL; M.NLp = I.NL; M.P = I.P; M.DAY = I.DAY;
    RunView R;
    int32_t *p = st;
    R.succ = p; p += S;
    R.pred = p; p += S;
    R.veh = p; p += S;
    R.endc = p; p += S;
    R.depc = p; p += S;
    R.inc = p; p += S;
    R.svco = p; p += S;
    int32_t *pick_w = p; R.pick_s = p; p += S;
    int32_t *w_w = p; R.w_s = p; p += S;
    R.F = p; p += V;
    int32_t *order = p; p += n;
    if (NW) { R.arr = p; p += S; R.sl = p; p += S; R.pos = p; p += S; R.slp = p; p += S; }
    else { R.arr = R.sl = R.pos = R.slp = nullptr; }
    R.E = nullptr;

    // ---- empty schedule ----------------------------------------------------
    for (int x = lane; x < S; x += 32) {
        R.succ[x] = x;
        R.pred[x] = x;
        if (x < n) {
            R.veh[x] = -1;
            pick_w[x] = I.pick[x];
            w_w[x] = I.w[x];
            R.endc[x] = R.depc[x] = R.inc[x] = R.svco[x] = 0;
        } else {
            R.veh[x] = x - n;
            pick_w[x] = I.vloc[x - n];
            w_w[x] = I.DAY;
        }
    }
    for (int i = lane; i < n; i += 32) order[i] = G.base_order[i];
    __syncwarp();
    for (int v = lane; v < V; v += 32) {
        if (NW) nw_refresh_route(M, R, v);
        else refresh_slot(M, R, n + v);
        R.F[v] = 0;
    }
    // ---- seeded phase permutations (reading #41) -----------------------------
    const uint64_t seed = G.seeds ? G.seeds[run] : 0ull;
    if (lane == 0 && seed != 0) {
        int n0 = 0;
        for (int m = 0; m < n; m++) n0 += I.heli[m] != 0;
        uint64_t s = seed;
        const int lo[2] = {0, n0}, hi[2] = {n0, n};
        for (int ph = 0; ph < 2; ph++)
            for (int x = hi[ph] - 1; x >= lo[ph] + 1; x--) {
                int y = lo[ph] + (int)(splitmix64_next(s) % (uint64_t)(x - lo[ph] + 1));
                int t = order[x]; order[x] = order[y]; order[y] = t;
            }
    }
    __syncwarp();

    // ---- placement loop ------------------------------------------------------
    int status = AS_OK, repairs = 0;
    const uint64_t Nmoves = (uint64_t)n * (uint64_t)S + (uint64_t)n * (uint64_t)n;
    for (int i = 0; i < n; i++) {
        const int m = order[i];
        const int wm = w_w[m], hm = M.hl(m), pm = pick_w[m], dm = M.dl(m);
        bool placed = false;
        for (int attempt = 0; attempt < 2 && !placed; attempt++) {
            uint64_t kmin = KEY_NONE;
            for (int v = lane; v < V; v += 32) {
                const int c = M.cls(v);
                if (hm && !M.hok(c)) continue;                                  // lines 10-12
                const int term = n + v;
                int next = term;
                if (G.insert_mode == 1) {
                    int x = R.succ[term];
                    while (x < n && w_w[x] <= wm) x = R.succ[x];
                    next = x;
                }
                const int d_in = Tget(M, c, R.endc[next], pm) + M.sv(c, m);   // prev -> m
                const int d_out = Tget(M, c, dm, pick_w[next]) + R.svco[next];  // m -> next
                const int inc = d_in + d_out - R.inc[next];
                bool ok;
                if (NW) {
                    const int Am = R.depc[next] + d_in;
                    ok = Am <= wm && Am + d_out - R.arr[next] <= R.sl[next];
                } else {
                    ok = R.depc[next] + d_in <= wm && wm + d_out <= w_w[next];  // lines 13-28
                }
                ok = ok && R.F[v] + inc <= I.P;                                  // lines 29-31
                if (ok) {
                    uint64_t k = ((uint64_t)(uint32_t)(inc + DELTA_BIAS) << 32) | (uint32_t)v;
                    kmin = k < kmin ? k : kmin;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                uint64_t u = __shfl_xor_sync(0xFFFFFFFFu, kmin, o);
                kmin = u < kmin ? u : kmin;
            }
            if (kmin != KEY_NONE) {
                if (lane == 0) {                                                 // line 40
                    const int v = (int)(uint32_t)kmin;
                    const int inc = (int)(kmin >> 32) - DELTA_BIAS;
                    const int term = n + v;
                    int next = term;
                    if (G.insert_mode == 1) {
                        int x = R.succ[term];
                        while (x < n && w_w[x] <= wm) x = R.succ[x];
                        next = x;
                    }
                    const int prev = R.pred[next];
                    R.succ[prev] = m; R.pred[m] = prev; R.succ[m] = next; R.pred[next] = m;
                    R.veh[m] = v;
                    if (NW) nw_refresh_route(M, R, v);
                    else { refresh_slot(M, R, m); refresh_slot(M, R, next); }
                    R.F[v] += inc;
                }
                __syncwarp();
                placed = true;
                break;
            }
            // no vehicle: repair (lines 36-37) unless nothing is assigned yet
            if (attempt == 1 || i == 0 || repairs >= G.max_repairs) break;
            uint64_t best = KEY_NONE;
            for (uint64_t idx = lane; idx < Nmoves; idx += 32) {
                MoveEval e = eval_index<NW>(M, R, (uint32_t)idx, 0xFu, 0);
                if (e.valid && e.feasible && e.delta < 0) {
                    uint64_t k = make_key(0, e.delta, (uint32_t)idx);
                    best = k < best ? k : best;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                uint64_t u = __shfl_xor_sync(0xFFFFFFFFu, best, o);
                best = u < best ? u : best;
            }
            if (best == KEY_NONE) break;
            if (lane == 0) {
                const uint32_t idx = key_idx(best);
                MoveEval e = eval_index<NW>(M, R, idx, 0xFu, 0);
                apply_move<NW>(M, R, idx, e, 0, 0, false);
            }
            __syncwarp();
            repairs++;
        }
        if (!placed) { status = AS_ERR_INIT_FAILED; break; }
    }

    // ---- output CSR ------------------------------------------------------------
    if (lane == 0) {
        int32_t *bp = G.ptr_out + (size_t)run * (V + 1);
        int32_t *bm = G.ms_out ? G.ms_out + (size_t)run * n : nullptr;
        int pos = 0;
        for (int v = 0; v < V; v++) {
            bp[v] = pos;
            if (status != AS_OK) continue;
            int x = R.succ[n + v];
            while (x < n) { if (bm) bm[pos] = x; pos++; x = R.succ[x]; }
        }
        bp[V] = pos;
        if (G.status_out) G.status_out[run] = status;
        if (G.nrep_out) G.nrep_out[run] = repairs;
    }
}

size_t greedy_smem_bytes(const DevInst &I, int warps, bool T_smem, bool state_smem) {
    size_t b = T_smem ? (((size_t)I.NC * I.NL * I.NL * 4 + 15) & ~(size_t)15) : 0;
    if (state_smem) b += (size_t)warps * greedy_state_words(I.n, I.V, I.no_wait != 0) * 4;
    return b;
}

size_t greedy_state_bytes(const DevInst &I) { return (size_t)greedy_state_words(I.n, I.V, I.no_wait != 0) * 4; }

cudaError_t launch_greedy(const DevInst &I, int n_starts, int insert_mode, int max_repairs, const uint64_t *seeds,
                          int32_t *order_scratch, int32_t *state_global, int warps, bool T_smem, bool state_smem,
                          int32_t *ptr_out, int32_t *ms_out, int32_t *status_out, int32_t *nrep_out, cudaStream_t st) {
    if (I.n > 0) {
        k_greedy_order<<<(I.n + 255) / 256, 256, 0, st>>>(I, order_scratch);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    GreedyArgs G;
    G.inst = I;
    G.n_starts = n_starts;
    G.insert_mode = insert_mode;
    G.max_repairs = max_repairs;
    G.T_smem = T_smem;
    G.state_smem = state_smem;
    G.warps = warps;
    G.seeds = seeds;
    G.base_order = order_scratch;
    G.state_global = state_global;
    G.ptr_out = ptr_out;
    G.ms_out = ms_out;
    G.status_out = status_out;
    G.nrep_out = nrep_out;
    const size_t smem = greedy_smem_bytes(I, warps, T_smem, state_smem);
    const int blocks = (n_starts + warps - 1) / warps;
    cudaError_t e;
    if (I.no_wait) {
        e = cudaFuncSetAttribute(k_greedy<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_greedy<true><<<blocks, warps * 32, smem, st>>>(G);
    } else {
        e = cudaFuncSetAttribute(k_greedy<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_greedy<false><<<blocks, warps * 32, smem, st>>>(G);
    }
    return cudaGetLastError();
}

}  // namespace airsched
