// kernels.cu -- sm_100a kernels of the move-evaluation and selection engine.
//
//   k_eval_dump     : as_eval_moves -- one thread per canonical index, writes
//                     delta/flags and reduces the selection key (parity tool).
//   k_search<TABU>  : persistent NS/TS loop, one run per CTA (as_tabu_run,
//                     as_nbhd_run, as_batch_run).  Per iteration: every warp
//                     scores tiles of moves (relocate rows: m warp-uniform,
//                     lanes stride the target slot; swap rows paired so every
//                     warp sees n items), reduces the packed 64-bit key by
//                     warp shuffle then through shared memory, and one thread
//                     applies the winner -- no host round-trip per iteration.
//
// DESIGN.md describes the layout and the roofline of each kernel.
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.cuh"
#include "launch.h"

namespace airsched {

__device__ __forceinline__ MissionView global_view(const DevInst &I) {
    MissionView M;
    M.T = I.T; M.del = I.del; M.heli = I.heli; M.svc = I.svc; M.vcls = I.vcls8; M.vloc = I.vloc;
    M.clsheli = I.cls_heli; M.n = I.n; M.V = I.V; M.NL = I.NL; M.NLp = I.NL; M.P = I.P; M.DAY = I.DAY;
    return M;
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t u = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = u < v ? u : v;
    }
    return v;
}

// ----------------------------------------------------------------------------
// State construction from CSR (shared by the dump path; the persistent kernel
// does the same in its prologue).  One CTA.
__global__ void k_build_state(DevInst I, const int32_t *ptr, const int32_t *ms, RunViewG G) {
    const int n = I.n, V = I.V, S = n + V;
    for (int x = threadIdx.x; x < S; x += blockDim.x) {
        if (x < n) {
            G.veh[x] = -1;
            G.succ[x] = x;
            G.pred[x] = x;
            G.pick_s[x] = I.pick[x];
            G.w_s[x] = I.w[x];
        } else {
            int v = x - n;
            G.veh[x] = v;
            G.pick_s[x] = I.vloc[v];
            G.w_s[x] = I.DAY;
        }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        int prev = n + v;
        for (int i = ptr[v]; i < ptr[v + 1]; i++) {
            int m = ms[i];
            G.veh[m] = v;
            G.succ[prev] = m;
            G.pred[m] = prev;
            prev = m;
        }
        G.succ[prev] = n + v;
        G.pred[n + v] = prev;
    }
    __syncthreads();
    MissionView M = global_view(I);
    RunView R;
    R.succ = G.succ; R.pred = G.pred; R.veh = G.veh; R.endc = G.endc; R.depc = G.depc; R.inc = G.inc;
    R.svco = G.svco; R.pick_s = G.pick_s; R.w_s = G.w_s; R.F = G.F; R.E = nullptr;
    R.arr = G.arr; R.sl = G.sl; R.pos = G.pos; R.slp = G.slp;
    for (int x = threadIdx.x; x < S; x += blockDim.x) {
        if (x < n && G.veh[x] < 0) {
            G.endc[x] = G.depc[x] = G.inc[x] = G.svco[x] = 0;
            if (I.no_wait) G.arr[x] = G.sl[x] = G.pos[x] = G.slp[x] = 0;
            continue;
        }
        if (!I.no_wait) refresh_slot(M, R, x);
    }
    if (I.no_wait)
        for (int v = threadIdx.x; v < V; v += blockDim.x) nw_refresh_route(M, R, v);
    __syncthreads();
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        int f = 0;
        int x = G.succ[n + v];
        while (x < n) { f += G.inc[x]; x = G.succ[x]; }
        f += G.inc[n + v];
        G.F[v] = f;
    }
}

// One thread per canonical index.  delta/flags nullable; best key via atomicMin.
template <bool TABU, bool NW>
__global__ void k_eval_dump(DevInst I, RunViewG G, int it, long long cur, long long best, uint32_t mask,
                            int32_t *delta_out, uint8_t *flags_out, unsigned long long *best_key, uint64_t N) {
    MissionView M = global_view(I);
    RunView R;
    R.succ = G.succ; R.pred = G.pred; R.veh = G.veh; R.endc = G.endc; R.depc = G.depc; R.inc = G.inc;
    R.svco = G.svco; R.pick_s = G.pick_s; R.w_s = G.w_s; R.F = G.F; R.E = TABU ? G.E : nullptr;
    R.arr = G.arr; R.sl = G.sl; R.pos = G.pos; R.slp = G.slp;
    uint64_t kmin = KEY_NONE;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < N;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        MoveEval e = eval_index<NW>(M, R, (uint32_t)idx, mask, it);
        uint8_t fl = 0;
        int cls = move_class<TABU>(e, cur, best);
        if (e.valid) {
            fl |= 1;
            if (e.feasible) fl |= 2;
            if (e.tabu) fl |= 4;
            if (cls == 0) fl |= 8;
            if (cls == 1) fl |= 16;
        }
        if (delta_out) delta_out[idx] = e.valid ? e.delta : 0;
        if (flags_out) flags_out[idx] = fl;
        if (cls >= 0) {
            uint64_t k = make_key(cls, e.delta, (uint32_t)idx);
            kmin = k < kmin ? k : kmin;
        }
    }
    kmin = warp_min_u64(kmin);
    if ((threadIdx.x & 31) == 0 && kmin != KEY_NONE) atomicMin(best_key, (unsigned long long)kmin);
}

// ----------------------------------------------------------------------------
// Persistent search kernel: one run per CTA.
struct SmemLayout {
    // byte offsets, 16-byte aligned
    int T, del, heli, svc, vcls, vloc, clsheli;
    int succ, pred, veh, endc, depc, inc, svco, pick_s, w_s, F, E, bsucc, arr, sl, pos, slp;
    int red, ctrl, total;
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline SmemLayout make_layout(int n, int V, int NL, int NC, bool T_smem, bool E_smem, bool nw) {
    SmemLayout L;
    int o = 0;
    const int S = n + V;
    L.T = T_smem ? o : -1;
    o = align16(o + (T_smem ? NC * NL * NL * 4 : 0));
    L.del = o; o = align16(o + n * 4);
    L.heli = o; o = align16(o + n);
    L.svc = o; o = align16(o + NC * n * 4);
    L.vcls = o; o = align16(o + V);
    L.vloc = o; o = align16(o + V * 4);
    L.clsheli = o; o = align16(o + NC);
    L.succ = o; o = align16(o + S * 4);
    L.pred = o; o = align16(o + S * 4);
    L.veh = o; o = align16(o + S * 4);
    L.endc = o; o = align16(o + S * 4);
    L.depc = o; o = align16(o + S * 4);
    L.inc = o; o = align16(o + S * 4);
    L.svco = o; o = align16(o + S * 4);
    L.pick_s = o; o = align16(o + S * 4);
    L.w_s = o; o = align16(o + S * 4);
    L.F = o; o = align16(o + V * 4);
    L.bsucc = o; o = align16(o + S * 4);
    L.arr = o; o = align16(o + (nw ? S * 4 : 0));
    L.sl = o; o = align16(o + (nw ? S * 4 : 0));
    L.pos = o; o = align16(o + (nw ? S * 4 : 0));
    L.slp = o; o = align16(o + (nw ? S * 4 : 0));
    L.E = E_smem ? o : -1;
    o = align16(o + (E_smem ? n * V * 4 : 0));
    L.red = o; o = align16(o + 32 * 8);
    L.ctrl = o; o = align16(o + 16 * 4);
    L.total = o;
    return L;
}

size_t search_smem_bytes(int n, int V, int NL, int NC, bool T_smem, bool E_smem, bool nw) {
    return (size_t)make_layout(n, V, NL, NC, T_smem, E_smem, nw).total;
}

template <bool TABU, bool NW>
__global__ void __launch_bounds__(1024) k_search(SearchArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const DevInst &I = A.inst;
    const int n = I.n, V = I.V, S = n + V, NC = I.NC;
    const int run = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const SmemLayout L = make_layout(n, V, I.NL, NC, A.T_smem, A.E_smem, NW);

    // ---- stage instance constants -----------------------------------------
#define SM32(off) reinterpret_cast<int32_t *>(smem_raw + (off))
#define SM8(off) reinterpret_cast<uint8_t *>(smem_raw + (off))
    if (A.T_smem) {
        const int4 *src = reinterpret_cast<const int4 *>(I.T);
        int4 *dst = reinterpret_cast<int4 *>(smem_raw + L.T);
        int nT = NC * I.NL * I.NL;
        for (int i = tid; i < nT / 4; i += blockDim.x) dst[i] = src[i];
        for (int i = (nT / 4) * 4 + tid; i < nT; i += blockDim.x) SM32(L.T)[i] = I.T[i];
    }
    for (int i = tid; i < n; i += blockDim.x) {
        SM32(L.del)[i] = I.del[i];
        SM8(L.heli)[i] = I.heli[i];
    }
    for (int i = tid; i < NC * n; i += blockDim.x) SM32(L.svc)[i] = I.svc[i];
    for (int i = tid; i < V; i += blockDim.x) {
        SM8(L.vcls)[i] = (uint8_t)I.vcls[i];
        SM32(L.vloc)[i] = I.vloc[i];
    }
    for (int i = tid; i < NC; i += blockDim.x) SM8(L.clsheli)[i] = I.cls_heli[i];

    MissionView M;
    M.del = SM32(L.del); M.heli = SM8(L.heli); M.svc = SM32(L.svc); M.vcls = SM8(L.vcls); M.vloc = SM32(L.vloc);
    M.clsheli = SM8(L.clsheli); M.T = A.T_smem ? SM32(L.T) : I.T;
    M.n = n; M.V = V; M.NL = I.NL; M.NLp = I.NL; M.P = I.P; M.DAY = I.DAY;
    int32_t *Eg = A.E_smem ? SM32(L.E) : (A.E_global ? A.E_global + (size_t)run * n * V : nullptr);
    RunView R;
    R.succ = SM32(L.succ); R.pred = SM32(L.pred); R.veh = SM32(L.veh); R.endc = SM32(L.endc); R.depc = SM32(L.depc);
    R.inc = SM32(L.inc); R.svco = SM32(L.svco); R.pick_s = SM32(L.pick_s); R.w_s = SM32(L.w_s); R.F = SM32(L.F);
    R.E = TABU ? Eg : nullptr;
    R.arr = SM32(L.arr); R.sl = SM32(L.sl); R.pos = SM32(L.pos); R.slp = SM32(L.slp);
    int32_t *bsucc = SM32(L.bsucc);
    unsigned long long *red = reinterpret_cast<unsigned long long *>(smem_raw + L.red);
    int32_t *ctrl = SM32(L.ctrl);   // 0: stop, 1: copy-best, 2: infeasible flag
    int32_t *pick_w = SM32(L.pick_s);
    int32_t *w_w = SM32(L.w_s);

    // ---- start schedule (CSR) -> linked lists ------------------------------
    const int32_t *ptr = A.start_ptr + (A.shared_start ? 0 : (size_t)run * (V + 1));
    const int32_t *ms = A.start_ms + (A.shared_start ? 0 : (size_t)run * n);
    for (int x = tid; x < S; x += blockDim.x) {
        if (x < n) {
            R.veh[x] = -1;
            pick_w[x] = I.pick[x];
            w_w[x] = I.w[x];
        } else {
            R.veh[x] = x - n;
            pick_w[x] = I.vloc[x - n];
            w_w[x] = I.DAY;
        }
    }
    if (tid < 16) ctrl[tid] = 0;
    if (Eg && TABU)
        for (int i = tid; i < n * V; i += blockDim.x) Eg[i] = -1;
    __syncthreads();
    for (int v = tid; v < V; v += blockDim.x) {
        int prev = n + v;
        int bad = 0;
        int lo = ptr[v], hi = ptr[v + 1];
        if (lo < 0 || hi < lo || hi > n) bad = 1;
        else
            for (int i = lo; i < hi; i++) {
                int m = ms[i];
                if (m < 0 || m >= n) { bad = 1; break; }
                if (atomicCAS(&R.veh[m], -1, v) != -1) { bad = 1; break; }
                R.succ[prev] = m;
                R.pred[m] = prev;
                prev = m;
            }
        R.succ[prev] = n + v;
        R.pred[n + v] = prev;
        if (bad) atomicOr(&ctrl[2], 1);
    }
    __syncthreads();
    for (int x = tid; x < S; x += blockDim.x) {
        if (x < n && R.veh[x] < 0) { atomicOr(&ctrl[2], 1); continue; }
        if (ctrl[2] || NW) continue;
        refresh_slot(M, R, x);
        // con7/con8 of the incoming link, con9 compatibility
        if (R.depc[x] + R.inc[x] > R.w_s[x]) atomicOr(&ctrl[2], 1);
        if (x < n && M.hl(x) && !M.hok(M.cls(R.veh[x]))) atomicOr(&ctrl[2], 1);
    }
    __syncthreads();
    if (NW && !ctrl[2]) {
        // no-wait: arrivals depend on the whole prefix -> one thread per route
        for (int v = tid; v < V; v += blockDim.x) {
            nw_refresh_route(M, R, v);
            int x = R.succ[n + v];
            for (;;) {
                if (R.arr[x] > R.w_s[x]) atomicOr(&ctrl[2], 1);
                if (x < n && M.hl(x) && !M.hok(M.cls(v))) atomicOr(&ctrl[2], 1);
                if (x >= n) break;
                x = R.succ[x];
            }
        }
        __syncthreads();
    }
    if (!ctrl[2])
        for (int v = tid; v < V; v += blockDim.x) {
            int f = 0;
            int x = R.succ[n + v];
            for (int guard = 0; x < n && guard <= n; guard++) { f += R.inc[x]; x = R.succ[x]; }
            f += R.inc[n + v];
            R.F[v] = f;
            if (f > I.P || x < n) atomicOr(&ctrl[2], 1);   // con6 (or a corrupt list)
        }
    __syncthreads();

    as_run_result *res = A.results ? A.results + run : nullptr;
    if (ctrl[2]) {
        if (tid == 0 && res) {
            res->best_obj = res->final_obj = res->start_obj = -1;
            res->best_iter = -1;
            res->iters_done = 0;
            res->stop_reason = AS_STOP_INFEASIBLE_START;
            res->kicks_applied = 0;
        }
        if (tid == 0 && A.best_ptr) {
            for (int v = 0; v <= V; v++) A.best_ptr[(size_t)run * (V + 1) + v] = 0;
        }
        return;
    }

    // ---- seeded kick (O12), one thread ---------------------------------------
    __shared__ long long s_cur, s_best, s_start;
    __shared__ int s_best_iter, s_kicks;
    if (tid == 0) {
        int kicks = 0;
        uint64_t seed = A.seeds ? A.seeds[run] : A.seed;
        if (seed != 0 && n > 0) {
            uint64_t s = seed;
            uint64_t Rb = (uint64_t)n * (uint64_t)S;
            for (int k = 0; k < A.kick; k++) {
                for (int tr = 0; tr < 64; tr++) {
                    uint32_t idx = (uint32_t)(splitmix64_next(s) % Rb);
                    MoveEval e = eval_index<NW>(M, R, idx, 0xFu, 0);
                    if (e.valid && e.feasible) {
                        apply_move<NW>(M, R, idx, e, 0, 0, false);
                        kicks++;
                        break;
                    }
                }
            }
        }
        long long c = 0;
        for (int v = 0; v < V; v++) c += R.F[v];
        s_cur = c;
        s_best = c;
        s_start = c;
        s_best_iter = -1;
        s_kicks = kicks;
        ctrl[1] = 1;
    }
    __syncthreads();

    // ---- main loop -----------------------------------------------------------
    const uint32_t mask = A.mask;
    const int nq = n / 2;   // swap row pairs (rows q and n-2-q)
    int it = 0;
    for (; it < A.max_iters; it++) {
        if (ctrl[1]) {
            for (int x = tid; x < S; x += blockDim.x) bsucc[x] = R.succ[x];
        }
        const long long cur = s_cur, best = s_best;
        uint64_t kmin = KEY_NONE;
        // relocate rows: m warp-uniform, lanes over target slots
        for (int m = warp; m < n; m += nwarps) {
            RelocRow r = reloc_row(M, R, m);
            if (r.a < 0) continue;
            const uint32_t base = (uint32_t)m * (uint32_t)S;
            for (int t = lane; t < S; t += 32) {
                MoveEval e = reloc_eval<NW>(M, R, r, m, t, mask, it);
                int cls = move_class<TABU>(e, cur, best);
                if (cls >= 0) {
                    uint64_t k = make_key(cls, e.delta, base + t);
                    kmin = k < kmin ? k : kmin;
                }
            }
        }
        // swap rows, paired: row q (n-1-q items) + row n-2-q (q+1 items)
        const uint32_t Rb = (uint32_t)n * (uint32_t)S;
        for (int q = warp; q < nq; q += nwarps) {
            const int qb = n - 2 - q;
            const int lenA = n - 1 - q;
            const int len = qb > q ? n : lenA;
            for (int j = lane; j < len; j += 32) {
                int m1, m2;
                if (j < lenA) { m1 = q; m2 = q + 1 + j; }
                else { m1 = qb; m2 = j; }
                MoveEval e = swap_eval<NW>(M, R, m1, m2, mask, it);
                int cls = move_class<TABU>(e, cur, best);
                if (cls >= 0) {
                    uint64_t k = make_key(cls, e.delta, Rb + (uint32_t)m1 * n + m2);
                    kmin = k < kmin ? k : kmin;
                }
            }
        }
        kmin = warp_min_u64(kmin);
        if (lane == 0) red[warp] = kmin;
        __syncthreads();
        uint64_t kc = KEY_NONE;
        if (warp == 0) kc = warp_min_u64(lane < nwarps ? red[lane] : KEY_NONE);   // CTA minimum by one warp
        if (tid == 0) {
            uint64_t k = kc;
            int stop = 0;
            if (k == KEY_NONE) stop = 2;                       // no feasible move
            else if (key_cls(k) == 1 && (!TABU || A.strict_tabu_stop)) stop = TABU ? 2 : 1;
            ctrl[1] = 0;
            if (stop) {
                ctrl[0] = stop;
            } else {
                uint32_t idx = key_idx(k);
                MoveEval e = eval_index<NW>(M, R, idx, mask, it);
                apply_move<NW>(M, R, idx, e, it, A.tenure, TABU);
                long long c = s_cur + e.delta;
                s_cur = c;
                if (c < s_best) {
                    s_best = c;
                    s_best_iter = it;
                    ctrl[1] = 1;
                }
                if (A.trace) {
                    as_trace_rec tr;
                    tr.cur = c;
                    tr.best = s_best;
                    tr.idx = idx;
                    tr.delta = e.delta;
                    tr.cls = key_cls(k);
                    tr.it = it;
                    A.trace[(size_t)run * A.max_iters + it] = tr;
                }
                if (A.digest && TABU) {
                    A.digest[(size_t)run * A.max_iters + it] = tabu_digest(R.E, n, V, it);
                }
            }
        }
        __syncthreads();
        if (ctrl[0]) break;
    }
    if (ctrl[1]) {
        for (int x = tid; x < S; x += blockDim.x) bsucc[x] = R.succ[x];
    }
    __syncthreads();
    if (tid == 0) {
        if (res) {
            res->start_obj = s_start;
            res->best_obj = s_best;
            res->final_obj = s_cur;
            res->best_iter = s_best_iter;
            res->iters_done = it;
            res->stop_reason = ctrl[0] ? ctrl[0] : AS_STOP_MAX_ITERS;
            res->kicks_applied = s_kicks;
        }
        if (A.best_ptr) {
            int32_t *bp = A.best_ptr + (size_t)run * (V + 1);
            int32_t *bm = A.best_ms + (size_t)run * n;
            int pos = 0;
            for (int v = 0; v < V; v++) {
                bp[v] = pos;
                int x = bsucc[n + v];
                while (x < n) { bm[pos++] = x; x = bsucc[x]; }
            }
            bp[V] = pos;
        }
    }
    if (A.tabu_out && TABU && Eg) {
        for (int i = tid; i < n * V; i += blockDim.x) A.tabu_out[(size_t)run * n * V + i] = Eg[i];
    }
}

// ----------------------------------------------------------------------------
// Host-side launchers (declared in launch.h).
cudaError_t launch_build_state(const DevInst &I, const int32_t *ptr, const int32_t *ms, RunViewG &G,
                               cudaStream_t st) {
    k_build_state<<<1, 256, 0, st>>>(I, ptr, ms, G);
    return cudaGetLastError();
}

template <bool TABU>
static void eval_dump_nw(const DevInst &I, const RunViewG &G, int blocks, int threads, int it, long long cur,
                         long long best, uint32_t mask, int32_t *delta, uint8_t *flags, unsigned long long *best_key,
                         uint64_t N, cudaStream_t st) {
    if (I.no_wait)
        k_eval_dump<TABU, true><<<blocks, threads, 0, st>>>(I, G, it, cur, best, mask, delta, flags, best_key, N);
    else
        k_eval_dump<TABU, false><<<blocks, threads, 0, st>>>(I, G, it, cur, best, mask, delta, flags, best_key, N);
}

cudaError_t launch_eval_dump(const DevInst &I, const RunViewG &G, int mode, int it, long long cur, long long best,
                             uint32_t mask, int32_t *delta, uint8_t *flags, unsigned long long *best_key,
                             uint64_t N, int n_sm, cudaStream_t st) {
    int threads = 256;
    uint64_t blocks64 = (N + threads - 1) / threads;
    int blocks = (int)(blocks64 < (uint64_t)n_sm * 8 ? blocks64 : (uint64_t)n_sm * 8);
    if (blocks < 1) blocks = 1;
    if (mode == 1) eval_dump_nw<true>(I, G, blocks, threads, it, cur, best, mask, delta, flags, best_key, N, st);
    else eval_dump_nw<false>(I, G, blocks, threads, it, cur, best, mask, delta, flags, best_key, N, st);
    return cudaGetLastError();
}

template <bool TABU, bool NW>
static cudaError_t launch_search_t(const SearchArgs &A, int n_runs, int threads, size_t smem, cudaStream_t st) {
    cudaError_t err = cudaFuncSetAttribute(k_search<TABU, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    k_search<TABU, NW><<<n_runs, threads, smem, st>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_search(const SearchArgs &A, int mode, int n_runs, int threads, size_t smem, cudaStream_t st) {
    const bool nw = A.inst.no_wait != 0;
    if (mode == 1)
        return nw ? launch_search_t<true, true>(A, n_runs, threads, smem, st)
                  : launch_search_t<true, false>(A, n_runs, threads, smem, st);
    return nw ? launch_search_t<false, true>(A, n_runs, threads, smem, st)
              : launch_search_t<false, false>(A, n_runs, threads, smem, st);
}

__global__ void k_svc(const int32_t *T, const int32_t *pick, const int32_t *del, int32_t *svc, int n, int NL, int NC) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * NC; i += gridDim.x * blockDim.x) {
        int c = i / n, m = i % n;
        svc[i] = T[((size_t)c * NL + pick[m]) * NL + del[m]];
    }
}

// Node-cost table of the global-table scorers: TD[c][x][t] = T_c[x][pick_t] + T_c[pick_t][del_t] for a
// mission t, T_c[x][base_v] for the END slot t = n + v (the host checked every entry fits 16 bits).
__global__ void k_build_td(const int32_t *T, const int32_t *pick, const int32_t *del, const int32_t *vloc,
                           uint16_t *TD, int n, int V, int NL, int NC) {
    const int S = n + V;
    const int64_t total = (int64_t)NC * NL * S;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(i % S), x = (int)((i / S) % NL), c = (int)(i / ((int64_t)S * NL));
        const int32_t *Tc = T + (int64_t)c * NL * NL;
        int v;
        if (t < n) v = Tc[(int64_t)x * NL + pick[t]] + Tc[(int64_t)pick[t] * NL + del[t]];
        else v = Tc[(int64_t)x * NL + vloc[t - n]];
        TD[i] = (uint16_t)v;
    }
}

cudaError_t launch_build_td(const int32_t *T, const int32_t *pick, const int32_t *del, const int32_t *vloc,
                            uint16_t *TD, int n, int V, int NL, int NC, cudaStream_t st) {
    k_build_td<<<1024, 256, 0, st>>>(T, pick, del, vloc, TD, n, V, NL, NC);
    return cudaGetLastError();
}

cudaError_t launch_svc(const int32_t *T, const int32_t *pick, const int32_t *del, int32_t *svc, int n, int NL, int NC,
                       cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_svc<<<(n * NC + 255) / 256, 256, 0, st>>>(T, pick, del, svc, n, NL, NC);
    return cudaGetLastError();
}

}  // namespace airsched
