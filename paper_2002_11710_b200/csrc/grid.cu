// grid.cu -- k_grid: ONE large instance on the whole GPU (configs C4, C5).
//
// Persistent cooperative kernel, one CTA per SM.  Every CTA holds a replica of
// the run state (slot records, links, route totals; the tabu matrix too when it
// fits) in shared memory; the travel-time table is staged in shared memory
// when it fits, otherwise read from an L2-resident padded copy.  Per iteration:
//   1. every warp scores its share of the tiles (score.cuh: relocate tiles,
//      top-aligned swap tiles, adjacent-swap tiles), reduces to one packed key
//      per CTA, and thread 0 folds it into a global key with atomicMin;
//   2. grid.sync();
//   3. every CTA reads the winning key and applies the same move to its own
//      replica (identical integer arithmetic => identical replicas); CTA 0 also
//      writes the trace and the best schedule.
// One grid barrier per iteration; the keys are triple-buffered so a CTA that
// races ahead into iteration it+1 never sees a slot that is still being read.
// The tabu matrix, when it lives in global memory, is written by every CTA with
// identical values, so each CTA's own reads after its apply are up to date.
#include <cooperative_groups.h>
#include <cuda/atomic>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdint>

#include "compact.cuh"
#include "engine.cuh"
#include "launch.h"
#include "score.cuh"

namespace cg = cooperative_groups;

constexpr int GRID_THREADS = airsched::GRID_WARPS * 32;
constexpr int GRID_SWT_MAX = 4096;   // compact swap tiles held as a table in shared memory (16 KB)
constexpr int GRID_PH_CTAS = 256;    // per-CTA phase records (AS_OPT_PHASE_TIMES)
constexpr int GRID_CL_MAX = 16;      // CTAs of the cluster mode (non-portable cluster size)

namespace airsched {

__host__ __device__ inline GridLayout grid_layout(int n, int V, int NL, int NC, int NLp, int tbytes, int ebytes,
                                                  bool T_smem, bool E_smem, bool tabu, bool swap_rec, int G,
                                                  bool nw) {
    GridLayout L;
    const int S = n + V;
    int o = 0;
    L.T = o; o = al16(o + (T_smem ? NC * NL * NLp * tbytes : 0));
    L.CS = o; o = al16(o + S * 16);
    L.MH = o; o = al16(o + n);
    L.VC = o; o = al16(o + V * 4);
    L.CH = o; o = al16(o + NC);
    L.RS = o; o = al16(o + S * 16);
    L.LK = o; o = al16(o + S * 4);
    L.F = o; o = al16(o + V * 4);
    L.E = o; o = al16(o + (tabu && E_smem ? n * V * ebytes : 0));
    L.red = o; o = al16(o + 32 * 8 + 64);
    // compact swap tiles: the prefix over the row groups (nRG + 1 entries) and, when the list is short
    // (<= GRID_SWT_MAX tiles), the tile table itself (no search per tile).  G = 0: sized for any G (G = 1)
    const int Gs = G > 0 ? G : 1;
    const int nSC = n > 1 ? (n - 1 + 63) / 64 : 0, nRG = (n + Gs - 1) / Gs;
    int nst = 0;
    for (int g = 0; g < nRG && nst <= GRID_SWT_MAX; g++) nst += swap_chunks_of_group(n, nSC, Gs, g);
    L.RR = o; o = al16(o + (T_smem || nw ? 0 : n * 8));   // cached relocate rows (global-table FAST scorers)
    L.SP = o; o = al16(o + (nRG + 2) * 4);
    L.ST = o; o = al16(o + (nst <= GRID_SWT_MAX ? nst : 0) * 4);
    L.SR = o; o = al16(o + (swap_rec ? GRID_WARPS * 2 * SR_ROWS * 16 : 0));   // per-warp swap-row records
    L.NR = o; o = al16(o + (nw ? S * 16 : 0));   // no-wait: {arrival, suffix slack, position} per slot
    L.total = o;
    return L;
}

size_t grid_smem_bytes(int n, int V, int NL, int NC, int tbytes, int ebytes, bool T_smem, bool E_smem, bool tabu,
                       bool swap_rec, int G, bool nw) {
    return grid_layout(n, V, NL, NC, padded_stride(NL, tbytes), tbytes, ebytes, T_smem, E_smem, tabu, swap_rec, G,
                       nw).total;
}

__device__ __forceinline__ bool GT_spread(int ntiles, int nwarps_all) { return ntiles < nwarps_all; }

// Fused sharded run, one thread of CTA 0 per rank (after the grid minimum of this rank's tile
// slice is in gkey[q]): publish it to EVERY rank's symmetric window through the NVLink
// load/store mapping and fold the nranks slots of the local window into the all-ranks winner.
// A slot is {key, tag}: the key is stored first, then the tag (run epoch << 32 | iteration + 1)
// with a system-scope release; the reader spins on its local tags with acquire loads until
// every rank's tag for this iteration is there, then reads the keys.  No barrier object, no
// reset between runs (the epoch advances per call on every rank), no sentinel key values.
// Slots are triple-buffered by iteration: slot q is rewritten at it+3, which a peer reaches only
// after reading this rank's keys of it+1 and it+2, i.e. after this rank has read slot q.
// The wait is bounded (GridArgs::xr_timeout_ns of %globaltimer): a missing or dead peer makes
// the run stop with AS_STOP_COMM_ABORT (the host returns AS_ERR_COMM) instead of hanging.
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint64_t rank_exchange(const GridArgs &GA, int q, int it, uint64_t kl) {
    const int R = GA.xr_nranks;
    const unsigned long long tag = ((unsigned long long)GA.xr_epoch << 32) | (unsigned)(it + 1);
    const size_t off = (size_t)(q * R + GA.xr_rank) * 2 * sizeof(unsigned long long);
    for (int p = 0; p < R; p++) {
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(ncclGetLsaPointer(GA.xr_win, off, p));
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_system>(dst[0]).store(kl, cuda::memory_order_relaxed);
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_system>(dst[1]).store(tag, cuda::memory_order_release);
    }
    unsigned long long *mine = reinterpret_cast<unsigned long long *>(
        ncclGetLocalPointer(GA.xr_win, (size_t)q * R * 2 * sizeof(unsigned long long)));
    uint64_t kg = KEY_NONE;
    const uint64_t t0 = globaltimer_ns();
    for (int p = 0; p < R; p++) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> tg(mine[2 * p + 1]);
        while (tg.load(cuda::memory_order_acquire) != tag)
            if (globaltimer_ns() - t0 > GA.xr_timeout_ns) return KEY_ABORT;
        const uint64_t v = cuda::atomic_ref<unsigned long long, cuda::thread_scope_system>(mine[2 * p]).load(
            cuda::memory_order_relaxed);
        kg = v < kg ? v : kg;
    }
    return kg;
}

// TR: the table is read from global memory (row-local reads, score.cuh).
// The bookkeeping half of the apply (one thread): route totals, tabu expiries (and the transposed copy),
// objective, best-so-far, trace record.
template <bool TABU, class MV, class RV, class ET>
__device__ __forceinline__ void grid_bookkeeping(const SearchArgs &A, const GridArgs &GA, const MV &M, const RV &R, ET *Et,
                                                 uint32_t idx, int32_t delta, int cls, const MoveSplit &ms, int it,
                                                 int n, int S, long long &s_cur, long long &s_best, int &s_best_it,
                                                 int *ctrl) {
    move_totals(M, R, idx, ms, it, A.tenure, TABU);
    if (TABU && Et) {   // the transposed copy gets the same expiries (every CTA, identical values)
        const uint32_t Rb = (uint32_t)n * (uint32_t)S;
        if (idx < Rb) {
            Et[(size_t)ms.a * n + idx / S] = (ET)(it + A.tenure);
        } else {
            Et[(size_t)ms.a * n + (idx - Rb) / n] = (ET)(it + A.tenure);
            Et[(size_t)ms.b * n + (idx - Rb) % n] = (ET)(it + A.tenure);
        }
    }
    const long long c = s_cur + delta;
    s_cur = c;
    if (c < s_best) {
        s_best = c;
        s_best_it = it;
        ctrl[1] = 1;
    }
    if (blockIdx.x == 0 && A.trace) {
        as_trace_rec tr;
        tr.cur = c;
        tr.best = s_best;
        tr.idx = idx;
        tr.delta = delta;
        tr.cls = cls;
        tr.it = it;
        A.trace[it] = tr;
    }
}

// PH: the per-iteration phase timers (AS_OPT_PHASE_TIMES) -- a separate instantiation, because even
// untaken, their live accumulators cost the production kernel ~8 % on C1/C2/C4 (register pressure;
// profiles/r02/kgrid_phase_ab.jsonl).
// NW: the no-wait variant (f3, reading #40): every move by the engine's exact evaluation (general
// scorers), per-slot {arrival, suffix slack, position} records, whole-route refresh of the two changed routes.
// CL: the grid is ONE thread-block cluster (small instances, GridArgs::cluster): the per-iteration exchange is
// every CTA's key stored into every CTA's shared memory (DSMEM) and one cluster barrier, instead of a global
// atomicMin, a grid barrier and a global read (~0.3 instead of ~1.5 us per iteration).
template <bool TABU, class TT, class ET, bool FULL, bool TR, bool PH, bool NW = false, bool CL = false>
__global__ void __launch_bounds__(GRID_THREADS, 1) k_grid(SearchArgs A, GridArgs GA) {
    static_assert(!NW || (!FULL && !PH), "the no-wait variant runs the general scorers, without phase timers");
    static_assert(!CL || (!TR && !NW), "cluster mode: shared-memory tables, waiting model");
    extern __shared__ __align__(16) unsigned char smem[];
    cg::grid_group grid = cg::this_grid();
    const DevInst &I = A.inst;
    const int n = I.n, V = I.V, S = n + V, NC = I.NC, NL = I.NL, NLp = GA.NLp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const GridLayout L = GA.L;
    TT *Ts = GA.T_smem ? reinterpret_cast<TT *>(smem + L.T) : reinterpret_cast<TT *>(const_cast<void *>(GA.Tglobal));
    int4 *CS4 = reinterpret_cast<int4 *>(smem + L.CS);
    uint8_t *MH = smem + L.MH;
    uint32_t *VC = reinterpret_cast<uint32_t *>(smem + L.VC);
    uint8_t *CH = smem + L.CH;
    int4 *RS4 = reinterpret_cast<int4 *>(smem + L.RS);
    uint32_t *LK = reinterpret_cast<uint32_t *>(smem + L.LK);
    int32_t *F = reinterpret_cast<int32_t *>(smem + L.F);
    ET *E = TABU ? (GA.E_smem ? reinterpret_cast<ET *>(smem + L.E) : reinterpret_cast<ET *>(GA.Eglobal)) : nullptr;
    unsigned long long *red = reinterpret_cast<unsigned long long *>(smem + L.red);
    int *ctrl = reinterpret_cast<int *>(smem + L.red + 32 * 8);

    // ---- stage constants --------------------------------------------------
    if (GA.T_smem)
        for (int i = tid; i < NC * NL * NL; i += blockDim.x) {
            int c = i / (NL * NL), r = (i / NL) % NL, col = i % NL;
            Ts[(c * NL + r) * NLp + col] = (TT)I.T[i];
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

    CompactMV<TT> M;
    M.T = Ts; M.CS = reinterpret_cast<unsigned char *>(CS4); M.MH = MH; M.VC = VC; M.CH = CH;
    M.n = n; M.V = V; M.NL = NL; M.NLp = NLp; M.P = I.P; M.DAY = I.DAY;
    CompactRV<ET> R;
    unsigned char *RSb = reinterpret_cast<unsigned char *>(RS4);
    R.succ.base = reinterpret_cast<unsigned char *>(LK); R.pred.base = reinterpret_cast<unsigned char *>(LK);
    R.veh.base = RSb; R.endc.base = RSb; R.depc.base = RSb; R.inc.base = RSb; R.svco.base = RSb;
    R.pick_s.base = reinterpret_cast<unsigned char *>(CS4); R.w_s.base = reinterpret_cast<unsigned char *>(CS4);
    R.F = F; R.E = E;
    R.arr.base = R.sl.base = R.pos.base = R.slp.base = NW ? smem + L.NR : nullptr;

    // ---- start schedule -> replica (every CTA) -----------------------------
    for (int x = tid; x < S; x += blockDim.x) R.veh[x] = x < n ? (int16_t)-1 : (int16_t)(x - n);
    if (TABU && (GA.E_smem || blockIdx.x == 0))
        for (int i = tid; i < n * V; i += blockDim.x) E[i] = (ET)-1;
    if (TABU && !GA.E_smem && blockIdx.x == 0)
        for (int i = tid; i < n * V; i += blockDim.x) reinterpret_cast<ET *>(GA.Etglobal)[i] = (ET)-1;
    if (tid == 0) ctrl[0] = ctrl[1] = 0;
    __syncthreads();
    const int32_t *ptr = A.start_ptr, *ms = A.start_ms;
    for (int v = tid; v < V; v += blockDim.x) {
        int prev = n + v;
        for (int i = ptr[v]; i < ptr[v + 1]; i++) {
            int m = ms[i];
            R.veh[m] = (int16_t)v;
            R.succ[prev] = (uint16_t)m;
            R.pred[m] = (uint16_t)prev;
            prev = m;
        }
        R.succ[prev] = (uint16_t)(n + v);
        R.pred[n + v] = (uint16_t)prev;
    }
    __syncthreads();
    if constexpr (NW) {   // whole routes: incoming links, arrivals, positions, suffix slacks (engine.cuh)
        for (int v = tid; v < V; v += blockDim.x) nw_refresh_route(M, R, v);
    } else {
        for (int x = tid; x < S; x += blockDim.x) refresh_slot(M, R, x);
    }
    __syncthreads();
    for (int v = tid; v < V; v += blockDim.x) {
        int f = 0, x = R.succ[n + v];
        for (int g = 0; x < n && g <= n; g++) { f += R.inc[x]; x = R.succ[x]; }
        F[v] = f + R.inc[n + v];
    }
    __syncthreads();

    // ---- seeded kick (identical in every CTA) ------------------------------
    __shared__ long long s_cur, s_best, s_start;
    __shared__ int s_best_it, s_kicks;
    __shared__ int s_ap[8];   // the applied move handed from warp 0 to warp 1: idx, delta, a, b, da, db, stop, class
    if (tid == 0) {
        int kicks = 0;
        if (A.seed != 0 && n > 0) {
            uint64_t s = A.seed;
            const uint64_t Rb = (uint64_t)n * (uint64_t)S;
            for (int k = 0; k < A.kick; k++)
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
        long long c = 0;
        for (int v = 0; v < V; v++) c += F[v];
        s_cur = s_best = s_start = c;
        s_best_it = -1;
        s_kicks = kicks;
    }
    __syncthreads();
    if (blockIdx.x == 0)
        for (int x = tid; x < S; x += blockDim.x) GA.BS[x] = (int32_t)(LK[x] & 0xFFFF);
    if constexpr (CL) cg::this_cluster().sync();
    else if (gridDim.x > 1) grid.sync();   // global tabu matrix initialised before anyone reads it
    __shared__ unsigned long long s_ckey[2][GRID_CL_MAX];   // CL: every CTA's key of iterations of each parity
    __shared__ unsigned long long s_kcl;                     // CL: the cluster minimum

    ScoreCtx<TT, ET> SC;
    SC.Ts = Ts; SC.Tt = I.tsym ? Ts : reinterpret_cast<const TT *>(I.TpadT); SC.CS4 = CS4; SC.MH = MH; SC.VC = VC; SC.RS4 = RS4; SC.LK = LK; SC.F = F; SC.E = E;
    ET *Et = TABU && !GA.E_smem ? reinterpret_cast<ET *>(GA.Etglobal) : nullptr;
    SC.Et = Et;
    SC.TD = GA.T_smem ? nullptr : I.TDg;   // node costs for the global-table scorers
    // global table + FAST scorers: each CTA caches the relocate rows' removal side (one global-table read
    // and four dependent shared loads per row and target chunk otherwise); built here, refreshed for the
    // two changed routes after every apply
    int2 *RR = (TR && FULL) ? reinterpret_cast<int2 *>(smem + L.RR) : nullptr;
    if (RR) {
        for (int m = tid; m < n; m += blockDim.x) RR[m] = reloc_row_record(Ts, CS4, RS4, LK, VC, F, NL, NLp, I.P, m);
        __syncthreads();
    }
    SC.RR = RR;
    SC.SR = (TR && FULL && GA.swap_rec) ? reinterpret_cast<int4 *>(smem + L.SR) : nullptr;
    SC.n = n; SC.V = V; SC.S = S; SC.NL = NL; SC.NLp = NLp; SC.P = I.P; SC.Rb = (uint32_t)n * (uint32_t)S;
    SC.mask = A.mask;
    SC.one = A.one; SC.neg = -A.one;
    GridTiles GT = grid_tiles(n, V, GA.G);
    if (GA.compact) {   // single GPU: the swap tiles below the diagonal are left out of the list
        int *SP = reinterpret_cast<int *>(smem + L.SP);
        int *ST = reinterpret_cast<int *>(smem + L.ST);
        if (tid == 0) {
            int c = 0;
            for (int g = 0; g < GT.nRG; g++) { SP[g] = c; c += swap_chunks_of_group(n, GT.nSC, GT.G, g); }
            SP[GT.nRG] = c;
        }
        __syncthreads();
        GT.swp = SP;
        GT.n_swap = SP[GT.nRG];
        GT.n_total = GT.n_reloc + GT.n_swap + GT.nAdj;
        if (GT.n_swap <= GRID_SWT_MAX) {
            for (int g = tid; g < GT.nRG; g += blockDim.x)
                for (int j = 0; j < SP[g + 1] - SP[g]; j++) ST[SP[g] + j] = (g << 16) | j;
            __syncthreads();
            GT.swt = ST;
        }
    }
    // tile -> warp: CTA-major (consecutive tiles = the same row group on one CTA: the table rows
    // of that group are shared in L1) when the tiles fill the grid; spread over the CTAs first when
    // there are fewer tiles than warps, so every SM scores at most ~one tile (latency-bound sizes)
    const int nwarps_all = gridDim.x * nwarps;
    const int gwarp = GT_spread(GA.thi - GA.tlo, nwarps_all) ? warp * gridDim.x + blockIdx.x : blockIdx.x * nwarps + warp;
    const bool one = gridDim.x == 1;
    unsigned long long *gkey = GA.gkey;   // [3], all KEY_NONE at launch

    int it = 0;
    // per-iteration device latency by phase (AS_OPT_PHASE_TIMES): thread 0 of CTA 0 reads %globaltimer
    // at the phase boundaries -- its own tiles, waiting for the CTA's other warps, CTA reduction + grid
    // barrier (+ rank exchange), apply -- and the sums go to GA.phase_ns at the end
    const bool ph = PH && blockIdx.x == 0 && tid == 0;
    const bool phc = PH && tid == 0;   // every CTA: its own tile phase (loop top -> all its warps done)
    unsigned long long ph_sum[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, ph_t = 0, ph_u = 0, ph_v = 0, phc_t = 0, phc_sum = 0;
    for (; it < A.max_iters; it++) {
        const long long cur = s_cur, best = s_best;
        if (ph) ph_t = globaltimer_ns();
        if (phc) phc_t = globaltimer_ns();
        uint64_t kmin = score_tiles<TABU, FULL, TR, NW>(SC, M, R, GT, GA.tlo, GA.thi, gwarp, nwarps_all, it, cur, best,
                                                        lane);
        kmin = wmin(kmin);
        if (ph) { ph_u = globaltimer_ns(); ph_sum[0] += ph_u - ph_t; ph_t = ph_u; }
        if (lane == 0) red[warp] = kmin;
        __syncthreads();
        if (phc) phc_sum += globaltimer_ns() - phc_t;
        if (ph) { ph_u = globaltimer_ns(); ph_sum[1] += ph_u - ph_t; ph_t = ph_u; }
        uint64_t kcta = KEY_NONE;
        if (warp == 0) {   // CTA minimum by one warp (parallel loads + shuffles, not a serial loop)
            kcta = wmin(lane < nwarps ? red[lane] : KEY_NONE);
            if constexpr (CL) {   // lane r stores this CTA's key into CTA r's slot (DSMEM)
                if (lane < (int)gridDim.x) {
                    unsigned long long *dst = cg::this_cluster().map_shared_rank(&s_ckey[it & 1][blockIdx.x], lane);
                    *dst = kcta;
                }
            } else if (lane == 0 && !one) {
                if (kcta != KEY_NONE) atomicMin(&gkey[it % 3], (unsigned long long)kcta);
                if (blockIdx.x == 0) gkey[(it + 1) % 3] = KEY_NONE;   // safe: last read in iteration it-2
            }
        }
        if constexpr (CL) {
            // slots of parity it & 1: written before this barrier, read after it; the next writes of this
            // parity (iteration it + 2) come after every CTA passed the barrier of iteration it + 1
            cg::this_cluster().sync();
            if (warp == 0) {
                const uint64_t kc = wmin(lane < (int)gridDim.x ? s_ckey[it & 1][lane] : KEY_NONE);
                if (lane == 0) s_kcl = kc;
            }
            __syncwarp();
        } else if (!one) {
            grid.sync();   // a single CTA (small instances) needs no grid barrier
        }
        if (GA.xr) {   // fused sharded run: the all-ranks minimum over NVLink, then every CTA reads it
            if (blockIdx.x == 0 && tid == 0) {
                const int q = it % 3;
                const uint64_t kl = one ? kcta : __ldcg(&gkey[q]);
                GA.gkey2[q] = rank_exchange(GA, q, it, kl);
            }
            if (one) __syncthreads();
            else grid.sync();
        }
        if (ph) { ph_u = globaltimer_ns(); ph_sum[2] += ph_u - ph_t; ph_t = ph_u; }
        // apply (every CTA, identical arithmetic), on two warps: warp 0's lane 0 reads the key, tests the
        // stop conditions and splits the delta per route (the scorers proved the move valid and
        // feasible), hands (idx, delta, split) to warp 1 through shared memory and a named barrier, then
        // relinks; warp 0's lanes refresh the touched incoming-link records.  Meanwhile warp 1's lane 0
        // updates the route totals, the tabu matrix (and its transpose), the objective and the trace --
        // disjoint state, so the two halves overlap (the split has read everything they change).
        if (warp == 0) {
            int nt = 0;
            if (lane == 0) {
                const uint64_t k = CL ? s_kcl : GA.xr ? __ldcg(&GA.gkey2[it % 3]) : one ? kcta : __ldcg(&gkey[it % 3]);
                if (ph) { asm volatile("" ::"l"(k)); ph_sum[4] += globaltimer_ns() - ph_t; }   // key read (part of apply)
                int stop = 0;
                if (k == KEY_ABORT) stop = AS_STOP_COMM_ABORT;   // a peer never arrived (bounded wait)
                else if (k == KEY_NONE) stop = AS_STOP_NO_MOVE;
                else if (key_cls(k) == 1 && (!TABU || A.strict_tabu_stop)) stop = TABU ? AS_STOP_NO_MOVE : AS_STOP_LOCAL_OPT;
                ctrl[0] = stop;
                ctrl[1] = 0;
                MoveSplit ms{0, 0, 0, 0};
                const uint32_t idx = key_idx(k);
                const int32_t delta = key_delta(k);
                if (!stop) {
                    if (ph) ph_v = globaltimer_ns();
                    ms = move_split(M, R, idx, delta);
                    if (ph) { asm volatile("" ::"r"(ms.a), "r"(ms.da)); ph_u = globaltimer_ns(); ph_sum[5] += ph_u - ph_v; ph_v = ph_u; }
                }
                s_ap[0] = (int)idx; s_ap[1] = delta; s_ap[2] = ms.a; s_ap[3] = ms.b; s_ap[4] = ms.da; s_ap[5] = ms.db;
                s_ap[6] = stop; s_ap[7] = key_cls(k);
                __threadfence_block();
            }
            __syncwarp();
            if (nwarps > 1) asm volatile("bar.arrive 1, 64;" ::: "memory");   // hand the split to warp 1
            if (lane == 0 && !ctrl[0]) {
                const uint32_t idx = (uint32_t)s_ap[0];
                nt = move_relink(M, R, idx, s_ap[2], s_ap[3], ctrl + 4);
                if (ph) { asm volatile("" ::"r"(nt)); ph_u = globaltimer_ns(); ph_sum[6] += ph_u - ph_v; ph_v = ph_u; }
                if (nwarps == 1) {   // (a one-warp CTA does the bookkeeping itself)
                    const MoveSplit ms{s_ap[2], s_ap[3], s_ap[4], s_ap[5]};
                    grid_bookkeeping<TABU>(A, GA, M, R, Et, idx, s_ap[1], s_ap[7], ms, it, n, S, s_cur, s_best, s_best_it,
                                           ctrl);
                }
            }
            nt = __shfl_sync(0xFFFFFFFFu, nt, 0);
            __syncwarp();
            if constexpr (NW) {   // the two changed routes, one lane each (s_ap: routes a, b)
                if (!ctrl[0] && lane < 2 && (lane == 0 || s_ap[3] != s_ap[2])) nw_refresh_route(M, R, s_ap[2 + lane]);
            } else {
                if (lane < nt) refresh_slot(M, R, ctrl[4 + lane]);
            }
            __syncwarp();
            if (ph) { ph_u = globaltimer_ns(); ph_sum[8] += ph_u - ph_v; }
        } else if (warp == 1) {
            asm volatile("bar.sync 1, 64;" ::: "memory");   // the split is in s_ap
            if (lane == 0 && !s_ap[6]) {
                const MoveSplit ms{s_ap[2], s_ap[3], s_ap[4], s_ap[5]};
                grid_bookkeeping<TABU>(A, GA, M, R, Et, (uint32_t)s_ap[0], s_ap[1], s_ap[7], ms, it, n, S, s_cur, s_best,
                                       s_best_it, ctrl);
            }
        }
        __syncthreads();
        if (RR && !ctrl[0]) {   // the applied move changed routes a and b only: refresh their rows
            const int ra = s_ap[2], rb = s_ap[3];
            for (int m = tid; m < n; m += blockDim.x) {
                const int v = R.veh[m];
                if (v == ra || v == rb) RR[m] = reloc_row_record(Ts, CS4, RS4, LK, VC, F, NL, NLp, I.P, m);
            }
            __syncthreads();
        }
        if (ph) ph_sum[3] += globaltimer_ns() - ph_t;
        if (ctrl[0]) break;
        if (ctrl[1] && blockIdx.x == 0)
            for (int x = tid; x < S; x += blockDim.x) GA.BS[x] = (int32_t)(LK[x] & 0xFFFF);
    }
    if (PH && phc && blockIdx.x < GRID_PH_CTAS) {   // per CTA: tile-phase sum and the SM it ran on
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        GA.phase_ns[16 + blockIdx.x] = phc_sum;
        GA.phase_ns[16 + GRID_PH_CTAS + blockIdx.x] = smid;
    }
    if (PH && ph) {
        for (int k = 0; k < 4; k++) GA.phase_ns[k] = ph_sum[k];
        GA.phase_ns[4] = (unsigned long long)it;
        GA.phase_ns[5] = ph_sum[4];
        for (int k = 5; k < 9; k++) GA.phase_ns[k + 1] = ph_sum[k];
    }
    if (blockIdx.x == 0 && tid == 0) {
        as_run_result *res = A.results;
        if (res) {
            res->start_obj = s_start;
            res->best_obj = s_best;
            res->final_obj = s_cur;
            res->best_iter = s_best_it;
            res->iters_done = it;
            res->stop_reason = ctrl[0] ? ctrl[0] : AS_STOP_MAX_ITERS;
            res->kicks_applied = s_kicks;
        }
    }
    if (blockIdx.x == 0 && A.tabu_out && TABU)
        for (int i = tid; i < n * V; i += blockDim.x) A.tabu_out[i] = (int32_t)E[i];
}

// Best schedule (global BS successor array) -> CSR; one thread.
__global__ void k_bs_to_csr(const int32_t *BS, int n, int V, int32_t *bp, int32_t *bm) {
    if (threadIdx.x || blockIdx.x) return;
    int pos = 0;
    for (int v = 0; v < V; v++) {
        bp[v] = pos;
        int x = BS[n + v];
        for (int g = 0; x < n && g < n; g++) { bm[pos++] = x; x = BS[x]; }
    }
    bp[V] = pos;
}

// Launch configuration of the cluster mode (one cluster of cl CTAs); gridDim.x == 0 on error.
static cudaLaunchConfig_t cluster_config(const void *kc, int cl, int threads, size_t smem, cudaStream_t st,
                                         cudaLaunchAttribute *at) {
    cudaLaunchConfig_t cfg = {};
    cudaError_t err = cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess && cl > 8) err = cudaFuncSetAttribute(kc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return cfg;
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
}

// How many clusters of cl CTAs of the cluster-mode kernel for (mode, table and tabu widths, FAST scorers) fit
// the GPU at once (0: none -- the caller keeps the cooperative grid).
int grid_cluster_capacity(int mode, int tbytes, int ebytes, bool full, int cl, int threads, size_t smem) {
    if (cl < 2 || cl > GRID_CL_MAX) return 0;
    const int eb = mode == 1 && tbytes == 2 && ebytes == 2 ? 2 : 4;
    const void *kc;
    if (mode == 1) {
        if (tbytes == 2 && eb == 2)
            kc = full ? (const void *)k_grid<true, uint16_t, int16_t, true, false, false, false, true>
                      : (const void *)k_grid<true, uint16_t, int16_t, false, false, false, false, true>;
        else if (tbytes == 2)
            kc = full ? (const void *)k_grid<true, uint16_t, int32_t, true, false, false, false, true>
                      : (const void *)k_grid<true, uint16_t, int32_t, false, false, false, false, true>;
        else kc = (const void *)k_grid<true, int32_t, int32_t, false, false, false, false, true>;
    } else {
        if (tbytes == 2)
            kc = full ? (const void *)k_grid<false, uint16_t, int32_t, true, false, false, false, true>
                      : (const void *)k_grid<false, uint16_t, int32_t, false, false, false, false, true>;
        else kc = (const void *)k_grid<false, int32_t, int32_t, false, false, false, false, true>;
    }
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = cluster_config(kc, cl, threads, smem, 0, at);
    if (cfg.gridDim.x == 0) { cudaGetLastError(); return 0; }
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kc, &cfg) != cudaSuccess) { cudaGetLastError(); return 0; }
    return n;
}

template <bool TABU, class TT, class ET, bool FULL>
static cudaError_t launch_g(const SearchArgs &A, const GridArgs &GA, int blocks, int threads, size_t smem,
                            cudaStream_t st) {
    auto kern = GA.phase_ns ? (GA.T_smem ? k_grid<TABU, TT, ET, FULL, false, true> : k_grid<TABU, TT, ET, FULL, true, true>)
                            : (GA.T_smem ? k_grid<TABU, TT, ET, FULL, false, false> : k_grid<TABU, TT, ET, FULL, true, false>);
    if constexpr (!FULL)   // the no-wait variant (general scorers; no phase-timer instantiation)
        if (A.inst.no_wait)
            kern = GA.T_smem ? k_grid<TABU, TT, ET, false, false, false, true> : k_grid<TABU, TT, ET, false, true, false, true>;
    SearchArgs a = A;
    GridArgs g = GA;
    void *args[] = {&a, &g};
    if (GA.cluster > 1) {   // one cluster of GA.cluster CTAs (shared-memory tables, waiting model)
        const void *kc = GA.phase_ns ? (const void *)k_grid<TABU, TT, ET, FULL, false, true, false, true>
                                     : (const void *)k_grid<TABU, TT, ET, FULL, false, false, false, true>;
        cudaLaunchAttribute at[1];
        cudaLaunchConfig_t cfg = cluster_config(kc, GA.cluster, threads, smem, st, at);
        if (cfg.gridDim.x == 0) return cudaGetLastError();
        return cudaLaunchKernelExC(&cfg, kc, args);
    }
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    return cudaLaunchCooperativeKernel((void *)kern, blocks, threads, args, smem, st);
}

cudaError_t launch_grid(const SearchArgs &A, GridArgs GA, int mode, int tbytes, int blocks, int threads, size_t smem,
                        cudaStream_t st) {
    const DevInst &I = A.inst;
    GA.NLp = padded_stride(I.NL, tbytes);
    const int eb = mode == 1 && tbytes == 2 && GA.ebytes == 2 ? 2 : 4;   // int16 expiries: half the tabu traffic
    GA.L = grid_layout(I.n, I.V, I.NL, I.NC, GA.NLp, tbytes, eb, GA.T_smem, GA.E_smem, mode == 1, GA.swap_rec != 0,
                       GA.G, I.no_wait != 0);
    const bool full = (A.mask & 15u) == 15u && A.inst.svcpos && !A.inst.no_wait;
    cudaError_t err;
    if (mode == 1) {
        if (tbytes == 2 && eb == 2)
            err = full ? launch_g<true, uint16_t, int16_t, true>(A, GA, blocks, threads, smem, st)
                       : launch_g<true, uint16_t, int16_t, false>(A, GA, blocks, threads, smem, st);
        else if (tbytes == 2) err = full ? launch_g<true, uint16_t, int32_t, true>(A, GA, blocks, threads, smem, st)
                                         : launch_g<true, uint16_t, int32_t, false>(A, GA, blocks, threads, smem, st);
        else err = launch_g<true, int32_t, int32_t, false>(A, GA, blocks, threads, smem, st);
    } else {
        if (tbytes == 2) err = full ? launch_g<false, uint16_t, int32_t, true>(A, GA, blocks, threads, smem, st)
                                    : launch_g<false, uint16_t, int32_t, false>(A, GA, blocks, threads, smem, st);
        else err = launch_g<false, int32_t, int32_t, false>(A, GA, blocks, threads, smem, st);
    }
    if (err != cudaSuccess) return err;
    if (A.best_ptr) {
        k_bs_to_csr<<<1, 1, 0, st>>>(GA.BS, I.n, I.V, A.best_ptr, A.best_ms);
        err = cudaGetLastError();
    }
    return err;
}

__global__ void k_pad_table(const int32_t *T, void *out, int NC, int NL, int NLp, int tbytes, int transpose) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < NC * NL * NL; i += gridDim.x * blockDim.x) {
        int c = i / (NL * NL), r = (i / NL) % NL, col = i % NL;
        size_t o = transpose ? (size_t)(c * NL + col) * NLp + r : (size_t)(c * NL + r) * NLp + col;
        if (tbytes == 2) reinterpret_cast<uint16_t *>(out)[o] = (uint16_t)T[i];
        else reinterpret_cast<int32_t *>(out)[o] = T[i];
    }
}

cudaError_t launch_pad_table(const int32_t *T, void *out, int NC, int NL, int NLp, int tbytes, bool transpose,
                             cudaStream_t st) {
    k_pad_table<<<256, 256, 0, st>>>(T, out, NC, NL, NLp, tbytes, transpose ? 1 : 0);
    return cudaGetLastError();
}

int padded_stride_host(int NL, int tbytes) { return padded_stride(NL, tbytes); }

}  // namespace airsched
