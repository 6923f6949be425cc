// batch.cu -- k_batch: many independent NS/TS runs, ONE RUN PER WARP.
//
// Design (profiles/r01/README.md): a CTA holds RPC runs (one per
// warp) and one copy of the instance in shared memory (uint16 travel times when
// they fit, rows padded to an odd number of 32-bit words so column gathers
// spread over the banks).  A warp is a complete run executor: it scores the
// whole neighbourhood of its run, reduces the packed key with shuffles, and
// its lane 0 applies the winner -- no CTA barrier inside the iteration loop,
// so the serial apply of one run overlaps the scoring of the other runs on the
// SM.  The target-slot side of the relocate block and the m2 side of the swap
// block are cached in registers per 32-lane chunk and reused across every
// row, leaving ~3 shared-memory gathers per relocate move.
//
// State is array-of-structs so one LDS.128 fetches a slot's whole record:
//   CS[x] (CTA-wide, 16 B): {w, pick | del << 16, svc_class0, svc_class1}
//   RS[x] (per run, 16 B):  {depc, inc, svco, endc | veh << 16}
//   LK[x] (per run, 4 B):   {succ | pred << 16}
// The arithmetic is engine.cuh's (used here for the kick and the apply),
// rewritten for register-resident operands in the scoring loops.
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.cuh"
#include "launch.h"
#include "score.cuh"
#include "compact.cuh"
#include "window.cuh"

namespace airsched {

constexpr int MAXTHREADS = 896;    // <= 28 runs per CTA (one wave of 4096 runs on 148 SMs)

// win: the WINDOW scorers (window.cuh) -- the tabu matrix lives in global memory, the run block
// holds the tabu bits TB[n], the ring of the last tenure + 1 iterations' tabu writes and the
// warp's window buffer instead.
__host__ __device__ inline BatchLayout batch_layout(int n, int V, int NL, int NC, int tbytes, int ebytes, bool tabu,
                                                   bool win = false, int tenure = 0, bool tsym = true, bool nw = false) {
    BatchLayout L;
    const int S = n + V;
    const int NLp = padded_stride(NL, tbytes);
    int o = 0;
    L.T = o; o = al16(o + NC * NL * NLp * tbytes);
    L.CS = o; o = al16(o + S * 16);
    L.MH = o; o = al16(o + n);
    L.VC = o; o = al16(o + V * 4);
    L.CH = o; o = al16(o + NC);
    L.TT = o; o = al16(o + (win && !tsym ? NC * NL * NLp * tbytes : 0));   // transposed table (window scorers)
    // node costs d_c(x, t) (window scorers); 128 B of guard before them: the lowest swap chunk's
    // lanes with m2 < 0 (masked) form addresses up to 126 B before a TD row (window.cuh ya_base)
    if (win) o = al16(o + 128);
    L.TD = o; o = al16(o + (win ? NC * td_layer(n + V, NL) * 2 : 0));
    L.TDT = o; o = al16(o + (win ? NC * n * padded_stride(NL, 2) * 2 : 0)); // the same, [c][m][x]
    L.shared_bytes = o;
    int r = 0;
    L.RS = r; r = al16(r + S * 16);
    L.LK = r; r = al16(r + S * 4);
    L.BS = r; r = al16(r + S * 2);
    L.F = r; r = al16(r + V * 4);
    L.E = r; r = al16(r + (tabu && !win ? n * V * ebytes : 0));
    L.PM = r; r = al16(r + (win ? 0 : V * 2));
    L.SN = r; r = al16(r + (win ? 0 : n * 2));
    L.TB = r; r = al16(r + (win && tabu ? n * 4 : 0));
    L.RG = r; r = al16(r + (win && tabu ? 2 * (tenure + 1) * 4 : 0));
    L.WB = r; r = al16(r + (win ? WIN_ROWS * WIN_REC_INT4 * 16 : 0));
    L.NR = r; r = al16(r + (nw ? S * 16 : 0));
    L.run_bytes = r;
    return L;
}

void batch_smem(int n, int V, int NL, int NC, int tbytes, int ebytes, bool tabu, size_t *shared_bytes,
                size_t *run_bytes, bool win, int tenure, bool tsym, bool nw) {
    BatchLayout L = batch_layout(n, V, NL, NC, tbytes, ebytes, tabu, win, tenure, tsym, nw);
    *shared_bytes = L.shared_bytes;
    *run_bytes = L.run_bytes;
}

// One CTA of the batched executor: stage A.inst, then run this CTA's runs
// cta_run0 .. cta_run0 + RPC - 1 (one per warp; A's per-run arrays are indexed by
// that run number).
template <bool TABU, class TT, class ET, bool FULL, bool WIN, bool NW = false>
__device__ __forceinline__ void batch_cta(const SearchArgs &A, int RPC, const BatchLayout &L, int NLp, int cta_run0) {
    // WIN: the window scorers (every move kind); FULL then selects their positive-leg (svcpos) form.
    // NW: the no-wait variant (f3, reading #40) -- every move scored by the engine's exact
    // no-wait evaluation (arrival shifts against suffix slacks; intra-route stretches walked).
    static_assert(!WIN || (sizeof(TT) == 2 && sizeof(ET) == 4), "window scorers: uint16 table, int32 E");
    static_assert(!NW || (!WIN && !FULL), "the no-wait variant runs the general per-move evaluation");
    extern __shared__ __align__(16) unsigned char smem[];
    const DevInst &I = A.inst;
    const int n = I.n, V = I.V, S = n + V, NC = I.NC, NL = I.NL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    TT *Ts = reinterpret_cast<TT *>(smem + L.T);
    unsigned char *CS = smem + L.CS;
    int4 *CS4 = reinterpret_cast<int4 *>(CS);
    uint8_t *MH = smem + L.MH;
    uint32_t *VC = reinterpret_cast<uint32_t *>(smem + L.VC);
    uint8_t *CH = smem + L.CH;

    // ---- stage the instance (whole CTA) --------------------------------------
    for (int i = tid; i < NC * NL * NL; i += blockDim.x) {
        int c = i / (NL * NL), r = (i / NL) % NL, col = i % NL;
        Ts[(c * NL + r) * NLp + col] = (TT)I.T[i];
        if (WIN && !I.tsym) reinterpret_cast<TT *>(smem + L.TT)[(c * NL + col) * NLp + r] = (TT)I.T[i];
    }
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
        CS4[x] = r;
    }
    for (int i = tid; i < n; i += blockDim.x) MH[i] = I.heli[i];
    for (int i = tid; i < V; i += blockDim.x) {
        int c = I.vcls8[i];
        VC[i] = (uint32_t)c | ((uint32_t)I.cls_heli[c] << 8) | ((uint32_t)I.vloc[i] << 16);
    }
    for (int i = tid; i < NC; i += blockDim.x) CH[i] = I.cls_heli[i];
    if (WIN) {   // node costs d_c(x, m) = T_c[x][pick_m] + T_c[pick_m][del_m] (O2), uint16 (tdmax checked on the host)
        // TD over every slot t (END_v: T_c[x][base_v], no service leg), class layers td_layer apart
        const int NTDp = padded_stride(S, 2), LTD = td_layer(S, NL);
        uint16_t *TD = reinterpret_cast<uint16_t *>(smem + L.TD);
        for (int i = tid; i < NC * NL * S; i += blockDim.x) {
            const int c = i / (NL * S), x = (i / S) % NL, t = i % S;
            const int pt = t < n ? I.pick[t] : I.vloc[t - n];
            const uint16_t d = (uint16_t)(I.T[(c * NL + x) * NL + pt] + (t < n ? I.svc[c * n + t] : 0));
            TD[c * LTD + x * NTDp + t] = d;
            if (t < n) reinterpret_cast<uint16_t *>(smem + L.TDT)[(c * n + t) * padded_stride(NL, 2) + x] = d;
        }
    }
    __syncthreads();

    const int run = cta_run0 + warp;
    if (warp >= RPC || run >= A.n_runs) return;

    unsigned char *rb = smem + L.shared_bytes + warp * L.run_bytes;
    unsigned char *RSb = rb + L.RS;
    int4 *RS4 = reinterpret_cast<int4 *>(RSb);
    uint32_t *LK = reinterpret_cast<uint32_t *>(rb + L.LK);
    uint16_t *BS = reinterpret_cast<uint16_t *>(rb + L.BS);
    int32_t *F = reinterpret_cast<int32_t *>(rb + L.F);
    // tabu expiry matrix: shared memory, or (window scorers) this run's block of E_global
    ET *E = TABU ? (WIN ? reinterpret_cast<ET *>(A.E_global + (size_t)run * n * V) : reinterpret_cast<ET *>(rb + L.E))
                 : nullptr;
    uint32_t *TB = WIN && TABU ? reinterpret_cast<uint32_t *>(rb + L.TB) : nullptr;   // tabu bits (window.cuh)
    uint32_t *RG = WIN && TABU ? reinterpret_cast<uint32_t *>(rb + L.RG) : nullptr;   // tabu-write ring

    CompactMV<TT> M;
    M.T = Ts; M.CS = CS; M.MH = MH; M.VC = VC; M.CH = CH;
    M.n = n; M.V = V; M.NL = NL; M.NLp = NLp; M.P = I.P; M.DAY = I.DAY;
    CompactRV<ET> R;
    R.succ.base = rb + L.LK; R.pred.base = rb + L.LK;
    R.veh.base = RSb; R.endc.base = RSb; R.depc.base = RSb; R.inc.base = RSb; R.svco.base = RSb;
    R.pick_s.base = CS; R.w_s.base = CS;
    R.arr.base = R.sl.base = R.pos.base = R.slp.base = NW ? rb + L.NR : nullptr;
    R.F = F; R.E = E;
    CompactRV<ET> R0 = R;   // evaluation view: the window path takes tabu from TB, not from E in global memory
    if (WIN) R0.E = nullptr;

    // ---- start schedule (CSR) -> linked lists --------------------------------
    const int32_t *ptr = A.start_ptr + (A.shared_start ? 0 : (size_t)run * (V + 1));
    const int32_t *ms = A.start_ms + (A.shared_start ? 0 : (size_t)run * n);
    for (int x = lane; x < S; x += 32) R.veh[x] = x < n ? (int16_t)-1 : (int16_t)(x - n);
    if (TABU)
        for (int i = lane; i < n * V; i += 32) E[i] = (ET)-1;
    if (WIN && TABU) {
        for (int i = lane; i < n; i += 32) TB[i] = 0u;
        for (int i = lane; i < 2 * (A.tenure + 1); i += 32) RG[i] = 0xFFFFFFFFu;
    }
    __syncwarp();
    int bad = 0;
    if (ptr[V] != n || ptr[0] != 0) bad = 1;
    for (int v = lane; v < V && !bad; v += 32) {
        int lo = ptr[v], hi = ptr[v + 1];
        if (lo < 0 || hi < lo || hi > n) { bad = 1; break; }
        int prev = n + v;
        for (int i = lo; i < hi; i++) {
            int m = ms[i];
            if (m < 0 || m >= n) { bad = 1; break; }
            R.veh[m] = (int16_t)v;
            R.succ[prev] = (uint16_t)m;
            R.pred[m] = (uint16_t)prev;
            prev = m;
        }
        R.succ[prev] = (uint16_t)(n + v);
        R.pred[n + v] = (uint16_t)prev;
    }
    bad = __any_sync(0xFFFFFFFFu, bad);
    __syncwarp();
    if (!bad) {
        if constexpr (NW) {   // whole routes: arrivals, positions, suffix slacks (engine.cuh)
            for (int x = lane; x < n; x += 32)
                if (R.veh[x] < 0) bad = 1;                                          // unlisted => duplicate
            bad = __any_sync(0xFFFFFFFFu, bad);
            if (!bad)
                for (int v = lane; v < V; v += 32) nw_refresh_route(M, R, v);
            __syncwarp();
        }
        for (int x = lane; x < S && !bad; x += 32) {
            if (x < n && R.veh[x] < 0) { bad = 1; continue; }   // unlisted => a duplicate elsewhere
            if (!NW) refresh_slot(M, R, x);
            if (R.depc[x] + R.inc[x] > R.w_s[x]) bad = 1;                          // con7/con8 (no-wait: arrival)
            if (x < n && MH[x] && !M.hok(M.cls(R.veh[x]))) bad = 1;              // con9
        }
        bad = __any_sync(0xFFFFFFFFu, bad);
    }
    __syncwarp();
    if (!bad) {
        for (int v = lane; v < V; v += 32) {
            int f = 0, x = R.succ[n + v];
            for (int g = 0; x < n && g <= n; g++) { f += R.inc[x]; x = R.succ[x]; }
            f += R.inc[n + v];
            F[v] = f;
            if (f > I.P || x < n) bad = 1;                                        // con6
        }
        bad = __any_sync(0xFFFFFFFFu, bad);
    }
    as_run_result *res = A.results ? A.results + run : nullptr;
    if (bad) {
        if (lane == 0 && res) {
            res->best_obj = res->final_obj = res->start_obj = -1;
            res->best_iter = -1;
            res->iters_done = 0;
            res->stop_reason = AS_STOP_INFEASIBLE_START;
            res->kicks_applied = 0;
        }
        if (lane == 0 && A.best_ptr)
            for (int v = 0; v <= V; v++) A.best_ptr[(size_t)run * (V + 1) + v] = 0;
        return;
    }
    __syncwarp();

    // ---- seeded kick (O12), lane 0 -------------------------------------------
    int kicks = 0;
    if (lane == 0 && !A.sweep) {
        uint64_t seed = A.seeds ? A.seeds[run] : A.seed;
        if (seed != 0 && n > 0) {
            uint64_t s = seed;
            const uint64_t Rb = (uint64_t)n * (uint64_t)S;
            for (int k = 0; k < A.kick; k++)
                for (int tr = 0; tr < 64; tr++) {
                    uint32_t idx = (uint32_t)(splitmix64_next(s) % Rb);
                    MoveEval e = eval_index<NW>(M, R0, idx, 0xFu, 0);
                    if (e.valid && e.feasible) {
                        apply_move<NW>(M, R, idx, e, 0, 0, false);
                        kicks++;
                        break;
                    }
                }
        }
    }
    __syncwarp();
    long long cur = 0;
    for (int v = lane; v < V; v += 32) cur += F[v];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cur += __shfl_xor_sync(0xFFFFFFFFu, cur, o);
    const long long start = cur;
    long long best = cur;
    int best_it = -1;
    for (int x = lane; x < S; x += 32) BS[x] = (uint16_t)(LK[x] & 0xFFFF);

    const uint32_t mask = A.mask;
    const uint32_t Rb = (uint32_t)n * (uint32_t)S;
    ScoreCtx<TT, ET> SC;
    SC.Ts = Ts; SC.Tt = A.inst.tsym ? Ts : reinterpret_cast<const TT *>(A.inst.TpadT); SC.CS4 = CS4; SC.MH = MH; SC.VC = VC; SC.RS4 = RS4; SC.LK = LK; SC.F = F; SC.E = E; SC.Et = nullptr; SC.TD = nullptr; SC.RR = nullptr; SC.SR = nullptr;
    SC.n = n; SC.V = V; SC.S = S; SC.NL = NL; SC.NLp = NLp; SC.P = I.P; SC.Rb = Rb; SC.mask = mask;
    SC.one = A.one; SC.neg = A.neg;
    WinCtx W;
    W.WB = WIN ? reinterpret_cast<int4 *>(rb + L.WB) : nullptr;
    W.TB = TB;
    W.ttsm = (int)__cvta_generic_to_shared(WIN && !I.tsym ? (const void *)(smem + L.TT) : (const void *)Ts);
    W.tdsm = (int)__cvta_generic_to_shared(smem + L.TD);
    W.tdtsm = (int)__cvta_generic_to_shared(smem + L.TDT);
    W.NTDp = padded_stride(S, 2);
    W.LTD = td_layer(S, NL);
    const int ring = A.tenure + 1;
    int it = 0, stop = 0;
    if (A.sweep) {
        // ---- f1: the paper-literal (i, j) sweep of Alg. 2 / Alg. 3 (oracle or_sweep) ----
        uint16_t *PM = reinterpret_cast<uint16_t *>(rb + L.PM);
        uint16_t *SN = reinterpret_cast<uint16_t *>(rb + L.SN);
        uint64_t ps = A.seeds ? A.seeds[run] : A.seed;
        const bool shuffled = ps != 0;
        while (!stop && it < A.max_iters) {
            int moved = 0;
            if (lane == 0) {
                for (int v = 0; v < V; v++) PM[v] = (uint16_t)v;
                if (shuffled)
                    for (int x = V - 1; x >= 1; x--) {
                        const int y = (int)(splitmix64_next(ps) % (uint64_t)(x + 1));
                        const uint16_t tmp = PM[x]; PM[x] = PM[y]; PM[y] = tmp;
                    }
            }
            __syncwarp();
            for (int pi = 0; pi < V && !stop; pi++) {
                int Lr = 0;
                if (lane == 0) {
                    const int i = PM[pi];
                    for (int x = R.succ[n + i]; x < n && Lr < n; x = R.succ[x]) SN[Lr++] = (uint16_t)x;
                    if (shuffled)
                        for (int x = Lr - 1; x >= 1; x--) {
                            const int y = (int)(splitmix64_next(ps) % (uint64_t)(x + 1));
                            const uint16_t tmp = SN[x]; SN[x] = SN[y]; SN[y] = tmp;
                        }
                }
                Lr = bcast(Lr);
                __syncwarp();
                for (int jj = 0; jj < Lr; jj++) {
                    const int j = SN[jj];
                    const int asp = (int)(best - cur);
                    uint64_t kmin = KEY_NONE;
                    for (int t0 = 0; t0 < S; t0 += 32 * KR) {
                        const uint64_t kb = score_reloc<TABU, false>(SC, t0, j, j + 1, it, asp, lane);
                        kmin = kb < kmin ? kb : kmin;
                    }
                    kmin = wmin(kmin);
                    int improved = 0;
                    if (lane == 0) {
                        uint32_t idx = 0xFFFFFFFFu;
                        int32_t dl = 0;
                        if (kmin != KEY_NONE && key_cls(kmin) == 0) {     // CurrentMin not empty
                            idx = key_idx(kmin);
                            MoveEval e = eval_index(M, R, idx, mask, it);
                            apply_move(M, R, idx, e, it, A.tenure, TABU);
                            dl = e.delta;
                            cur += e.delta;
                            moved = 1;
                            if (cur < best) {
                                best = cur;
                                best_it = it;
                                improved = 1;
                            }
                        }
                        if (A.trace) {
                            as_trace_rec tr;
                            tr.cur = cur;
                            tr.best = best;
                            tr.idx = idx;
                            tr.delta = dl;
                            tr.cls = idx == 0xFFFFFFFFu ? -1 : 0;
                            tr.it = it;
                            A.trace[(size_t)run * A.max_iters + it] = tr;
                        }
                    }
                    cur = bcast(cur);
                    best = bcast(best);
                    improved = bcast(improved);
                    __syncwarp();
                    if (improved)
                        for (int x = lane; x < S; x += 32) BS[x] = (uint16_t)(LK[x] & 0xFFFF);
                    if (++it >= A.max_iters) { stop = 0; break; }
                }
                if (it >= A.max_iters) break;
            }
            moved = bcast(moved);
            if (it >= A.max_iters) break;
            if (!moved) stop = TABU ? AS_STOP_NO_MOVE : AS_STOP_LOCAL_OPT;   // a sweep without a move
        }
    }
    for (; !A.sweep && it < A.max_iters; it++) {
        __syncwarp();
        uint64_t kmin = KEY_NONE;
        const int asp = (int)(best - cur);   // aspiration: cur + delta < best  <=>  delta < asp
        if (WIN && TABU) {
            // tabu bits in force at iteration it: drop the pairs written at it - 1 - tenure (E = it - 1)
            // unless a later iteration of the ring wrote the same pair again (O8)
            const int slot = it % ring;
            const uint32_t o0 = RG[2 * slot], o1 = RG[2 * slot + 1];
            if (o0 != 0xFFFFFFFFu) {
                bool h0 = false, h1 = false;
                for (int e = lane; e < 2 * ring; e += 32) {
                    if ((e >> 1) == slot) continue;
                    const uint32_t x = RG[e];
                    h0 |= x == o0;
                    h1 |= x == o1;
                }
                h0 = __any_sync(0xFFFFFFFFu, h0);
                h1 = __any_sync(0xFFFFFFFFu, h1);
                if (lane == 0) {
                    if (!h0) TB[o0 & 0xFFFF] &= ~(0x80000000u >> (o0 >> 16));
                    if (o1 != 0xFFFFFFFFu && !h1) TB[o1 & 0xFFFF] &= ~(0x80000000u >> (o1 >> 16));
                    RG[2 * slot] = RG[2 * slot + 1] = 0xFFFFFFFFu;
                }
                __syncwarp();
            }
        }

        if constexpr (NW) {
            // no-wait: every move by the engine's exact evaluation -- relocate rows (m warp-uniform,
            // lanes over target slots), then swap rows (lanes over m2 > m1); adjacent pairs included
            for (int m = 0; m < n; m++) {
                const RelocRow r = reloc_row(M, R0, m);
                if (r.a < 0) continue;
                for (int t = lane; t < S; t += 32) {
                    const MoveEval e = reloc_eval<true>(M, R0, r, m, t, mask, it);
                    const int cls = move_class<TABU>(e, cur, best);
                    if (cls >= 0) {
                        const uint64_t key = make_key(cls, e.delta, (uint32_t)m * (uint32_t)S + (uint32_t)t);
                        kmin = key < kmin ? key : kmin;
                    }
                }
            }
            for (int m1 = 0; m1 + 1 < n; m1++)
                for (int m2 = m1 + 1 + lane; m2 < n; m2 += 32) {
                    const MoveEval e = swap_eval<true>(M, R0, m1, m2, mask, it);
                    const int cls = move_class<TABU>(e, cur, best);
                    if (cls >= 0) {
                        const uint64_t key = make_key(cls, e.delta, Rb + (uint32_t)m1 * (uint32_t)n + (uint32_t)m2);
                        kmin = key < kmin ? key : kmin;
                    }
                }
        } else {
        // Per-lane best inside a tile (score.cuh); tiles merged through the 64-bit key.  The window scorers
        // with positive legs run their one-sign-bit form first (F1, window.cuh) and the exact form only when
        // that finds no admissible feasible move (class 1 or none: the by-default move, a local optimum)
        auto score_blocks = [&](auto f1) {
            constexpr bool F1 = decltype(f1)::value;
            uint64_t km = KEY_NONE;
            // ============================ relocate block ============================
            for (int t0 = 0; t0 < S; t0 += 32 * KR) {
                uint64_t kb;
                if constexpr (WIN) kb = score_reloc_win<TABU, FULL, F1>(SC, W, t0, 0, n, it, asp, lane);
                else kb = FULL ? score_reloc_fast<TABU>(SC, t0, 0, n, it, asp, lane)
                               : score_reloc<TABU, FULL>(SC, t0, 0, n, it, asp, lane);
                km = kb < km ? kb : km;
            }
            // ============================== swap block ==============================
            // m2 chunks of 32*KS aligned to the top (hi = n, n - 64, ...) so only the
            // lowest chunk is ragged; adjacent pairs are excluded there and scored exactly
            // by the generic three-link formula below.
            for (int hi = n; hi > 1; hi -= 32 * KS) {
                uint64_t kb;
                if constexpr (WIN) kb = score_swap_win<TABU, FULL, F1>(SC, W, hi, 0, hi - 1, it, asp, lane);
                else kb = FULL ? score_swap_fast<TABU>(SC, hi, 0, hi - 1, it, asp, lane)
                               : score_swap<TABU, FULL>(SC, hi, 0, hi - 1, it, asp, lane);
                km = kb < km ? kb : km;
            }
            return km;
        };
        constexpr bool F1 = WIN && FULL;
        {
            const uint64_t km = score_blocks(std::integral_constant<bool, F1>{});
            kmin = km < kmin ? km : kmin;
        }
        if constexpr (F1) {
            if (key_cls(wmin(kmin)) == 1) {   // warp-uniform: no admissible feasible move -- re-score exactly
                const uint64_t km = score_blocks(std::integral_constant<bool, false>{});
                kmin = km;
            }
        }
        // adjacent pairs (x, succ x): the exact three-link formula (engine.cuh)
        if (mask & 8u) {
            for (int x = lane; x < n; x += 32) {
                const int g = LK[x] & 0xFFFF;
                if (R.veh[x] < 0 || g >= n) continue;
                const int m1 = min(x, g), m2 = max(x, g);
                MoveEval e = swap_eval(M, R0, m1, m2, mask, it);
                if (WIN && TABU) {   // placed-into pairs (m1, veh m2), (m2, veh m1): the same route here
                    const int v = R.veh[x];
                    e.tabu = ((TB[m1] | TB[m2]) << v) >> 31;
                }
                const int cls = move_class<TABU>(e, cur, best);
                if (cls >= 0) {
                    const uint64_t key = make_key(cls, e.delta, Rb + (uint32_t)m1 * (uint32_t)n + (uint32_t)m2);
                    kmin = key < kmin ? key : kmin;
                }
            }
        }
        }   // !NW

        // ============================ select + apply ============================
        kmin = wmin(kmin);
        int improved = 0;
        if (lane == 0) {
            if (kmin == KEY_NONE) stop = AS_STOP_NO_MOVE;
            else if (key_cls(kmin) == 1 && (!TABU || A.strict_tabu_stop)) stop = TABU ? AS_STOP_NO_MOVE : AS_STOP_LOCAL_OPT;
            if (!stop) {
                const uint32_t idx = key_idx(kmin);
                MoveEval e = eval_index<NW>(M, R0, idx, mask, it);
                if (WIN && TABU) {
                    // the 'from' pairs this move writes (O8): relocate (m, veh m); swap (m1, veh m1), (m2, veh m2)
                    uint32_t p0, p1 = 0xFFFFFFFFu;
                    if (idx < Rb) {
                        const int m = idx / S;
                        p0 = (uint32_t)m | ((uint32_t)R.veh[m] << 16);
                    } else {
                        const int m1 = (idx - Rb) / n, m2 = (idx - Rb) % n;
                        p0 = (uint32_t)m1 | ((uint32_t)R.veh[m1] << 16);
                        p1 = (uint32_t)m2 | ((uint32_t)R.veh[m2] << 16);
                    }
                    const int slot = it % ring;
                    RG[2 * slot] = p0;
                    RG[2 * slot + 1] = p1;
                    if (A.tenure > 0) {   // E = it + tenure >= it + 1: tabu from the next iteration on
                        TB[p0 & 0xFFFF] |= 0x80000000u >> (p0 >> 16);
                        if (p1 != 0xFFFFFFFFu) TB[p1 & 0xFFFF] |= 0x80000000u >> (p1 >> 16);
                    }
                }
                apply_move<NW>(M, R, idx, e, it, A.tenure, TABU);
                cur += e.delta;
                if (cur < best) {
                    best = cur;
                    best_it = it;
                    improved = 1;
                }
                if (A.trace) {
                    as_trace_rec tr;
                    tr.cur = cur;
                    tr.best = best;
                    tr.idx = idx;
                    tr.delta = e.delta;
                    tr.cls = key_cls(kmin);
                    tr.it = it;
                    A.trace[(size_t)run * A.max_iters + it] = tr;
                }
            }
        }
        stop = bcast(stop);
        if (stop) break;
        cur = bcast(cur);
        best = bcast(best);
        improved = bcast(improved);
        __syncwarp();
        if (improved)
            for (int x = lane; x < S; x += 32) BS[x] = (uint16_t)(LK[x] & 0xFFFF);
    }
    __syncwarp();
    if (lane == 0) {
        if (res) {
            res->start_obj = start;
            res->best_obj = best;
            res->final_obj = cur;
            res->best_iter = best_it;
            res->iters_done = it;
            res->stop_reason = stop ? stop : AS_STOP_MAX_ITERS;
            res->kicks_applied = kicks;
        }
        if (A.best_ptr) {
            int32_t *bp = A.best_ptr + (size_t)run * (V + 1);
            int32_t *bm = A.best_ms + (size_t)run * n;
            int pos = 0;
            for (int v = 0; v < V; v++) {
                bp[v] = pos;
                int x = BS[n + v];
                for (int g = 0; x < n && g < n; g++) { bm[pos++] = x; x = BS[x]; }
            }
            bp[V] = pos;
        }
    }
    if (A.tabu_out && TABU)
        for (int i = lane; i < n * V; i += 32) A.tabu_out[(size_t)run * n * V + i] = (int32_t)E[i];
}

template <bool TABU, class TT, class ET, bool FULL, bool WIN, bool NW = false>
__global__ void __launch_bounds__(MAXTHREADS, 1) k_batch(SearchArgs A, int RPC, BatchLayout L, int NLp) {
    batch_cta<TABU, TT, ET, FULL, WIN, NW>(A, RPC, L, NLp, blockIdx.x * RPC);
}

// Several instances in one launch (as_batch_run_jobs): CTA b runs cta[b] = {job, first run
// of the job, runs} with that job's instance staged in its shared memory; the per-run
// output arrays are re-based to the CTA's first run.
template <bool TABU, class TT, class ET, bool FULL, bool WIN>
__global__ void __launch_bounds__(MAXTHREADS, 1) k_batch_jobs(SearchArgs A, const BatchJob *jobs, const int4 *cta) {
    const int4 c = cta[blockIdx.x];
    const BatchJob &J = jobs[c.x];
    SearchArgs B = A;
    const size_t r = (size_t)J.run0 + c.y;
    B.inst = J.inst;
    B.start_ptr = J.start_ptr;
    B.start_ms = J.start_ms;
    B.shared_start = 1;
    B.n_runs = c.z;
    B.seeds = A.seeds ? A.seeds + r : nullptr;
    B.results = A.results ? A.results + r : nullptr;
    B.best_ptr = A.best_ptr ? A.best_ptr + J.bp_off + (size_t)c.y * (J.inst.V + 1) : nullptr;
    B.best_ms = A.best_ms ? A.best_ms + J.bm_off + (size_t)c.y * J.inst.n : nullptr;
    B.E_global = A.E_global ? A.E_global + J.e_off + (size_t)c.y * J.inst.n * J.inst.V : nullptr;
    B.trace = A.trace ? A.trace + r * (size_t)A.max_iters : nullptr;
    B.digest = nullptr;
    B.tabu_out = nullptr;
    batch_cta<TABU, TT, ET, FULL, WIN>(B, J.RPC, J.L, J.NLp, 0);
}

template <bool TABU, class TT, class ET, bool FULL, bool WIN = false, bool NW = false>
static cudaError_t launch_one(const SearchArgs &A, int RPC, size_t smem, cudaStream_t st) {
    auto kern = k_batch<TABU, TT, ET, FULL, WIN, NW>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const DevInst &I = A.inst;
    BatchLayout L = batch_layout(I.n, I.V, I.NL, I.NC, (int)sizeof(TT), (int)sizeof(ET), TABU, WIN, A.tenure, I.tsym,
                                 NW);
    int NLp = padded_stride(I.NL, (int)sizeof(TT));
    int grid = (A.n_runs + RPC - 1) / RPC;
    kern<<<grid, RPC * 32, smem, st>>>(A, RPC, L, NLp);
    return cudaGetLastError();
}

template <bool TABU, class TT, class ET, bool FULL, bool WIN = false>
static cudaError_t launch_jobs_t(const SearchArgs &A, const BatchJob *jobs, const int4 *cta, int n_cta, int threads,
                                 size_t smem, cudaStream_t st) {
    auto kern = k_batch_jobs<TABU, TT, ET, FULL, WIN>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    kern<<<n_cta, threads, smem, st>>>(A, jobs, cta);
    return cudaGetLastError();
}

cudaError_t launch_batch_jobs(const SearchArgs &A, const BatchJob *jobs, const int4 *cta, int n_cta, int threads,
                              size_t smem, int mode, int tbytes, int ebytes, bool full, cudaStream_t st, bool win) {
    if (win) {   // window scorers: uint16 table, tabu matrix in global memory (int32); full = positive legs
        if (full)
            return mode == 1 ? launch_jobs_t<true, uint16_t, int32_t, true, true>(A, jobs, cta, n_cta, threads, smem, st)
                             : launch_jobs_t<false, uint16_t, int32_t, true, true>(A, jobs, cta, n_cta, threads, smem, st);
        return mode == 1 ? launch_jobs_t<true, uint16_t, int32_t, false, true>(A, jobs, cta, n_cta, threads, smem, st)
                         : launch_jobs_t<false, uint16_t, int32_t, false, true>(A, jobs, cta, n_cta, threads, smem, st);
    }
    if (mode == 1) {
        if (tbytes == 2 && ebytes == 2)
            return full ? launch_jobs_t<true, uint16_t, int16_t, true>(A, jobs, cta, n_cta, threads, smem, st)
                        : launch_jobs_t<true, uint16_t, int16_t, false>(A, jobs, cta, n_cta, threads, smem, st);
        if (tbytes == 2) return launch_jobs_t<true, uint16_t, int32_t, false>(A, jobs, cta, n_cta, threads, smem, st);
        return ebytes == 2 ? launch_jobs_t<true, int32_t, int16_t, false>(A, jobs, cta, n_cta, threads, smem, st)
                           : launch_jobs_t<true, int32_t, int32_t, false>(A, jobs, cta, n_cta, threads, smem, st);
    }
    if (tbytes == 2)
        return full ? launch_jobs_t<false, uint16_t, int16_t, true>(A, jobs, cta, n_cta, threads, smem, st)
                    : launch_jobs_t<false, uint16_t, int16_t, false>(A, jobs, cta, n_cta, threads, smem, st);
    return launch_jobs_t<false, int32_t, int16_t, false>(A, jobs, cta, n_cta, threads, smem, st);
}

BatchLayout batch_layout_host(int n, int V, int NL, int NC, int tbytes, int ebytes, bool tabu, bool win, int tenure,
                              bool tsym) {
    return batch_layout(n, V, NL, NC, tbytes, ebytes, tabu, win, tenure, tsym);
}

cudaError_t launch_batch(const SearchArgs &A, int mode, int RPC, int tbytes, int ebytes, size_t smem,
                         cudaStream_t st, bool win) {
    if (A.inst.no_wait) {   // f3: general evaluation, int32 expiries
        if (tbytes == 2)
            return mode == 1 ? launch_one<true, uint16_t, int32_t, false, false, true>(A, RPC, smem, st)
                             : launch_one<false, uint16_t, int32_t, false, false, true>(A, RPC, smem, st);
        return mode == 1 ? launch_one<true, int32_t, int32_t, false, false, true>(A, RPC, smem, st)
                         : launch_one<false, int32_t, int32_t, false, false, true>(A, RPC, smem, st);
    }
    const bool full = (A.mask & 15u) == 15u && A.inst.svcpos;
    if (win) {   // window scorers: uint16 table, tabu matrix in global memory (int32); positive legs or general
        if (A.inst.svcpos)
            return mode == 1 ? launch_one<true, uint16_t, int32_t, true, true>(A, RPC, smem, st)
                             : launch_one<false, uint16_t, int32_t, true, true>(A, RPC, smem, st);
        return mode == 1 ? launch_one<true, uint16_t, int32_t, false, true>(A, RPC, smem, st)
                         : launch_one<false, uint16_t, int32_t, false, true>(A, RPC, smem, st);
    }
    if (mode == 1) {
        if (tbytes == 2 && ebytes == 2)
            return full ? launch_one<true, uint16_t, int16_t, true>(A, RPC, smem, st)
                        : launch_one<true, uint16_t, int16_t, false>(A, RPC, smem, st);
        if (tbytes == 2) return launch_one<true, uint16_t, int32_t, false>(A, RPC, smem, st);
        return ebytes == 2 ? launch_one<true, int32_t, int16_t, false>(A, RPC, smem, st)
                           : launch_one<true, int32_t, int32_t, false>(A, RPC, smem, st);
    }
    if (tbytes == 2)
        return full ? launch_one<false, uint16_t, int16_t, true>(A, RPC, smem, st)
                    : launch_one<false, uint16_t, int16_t, false>(A, RPC, smem, st);
    return launch_one<false, int32_t, int16_t, false>(A, RPC, smem, st);
}

}  // namespace airsched
