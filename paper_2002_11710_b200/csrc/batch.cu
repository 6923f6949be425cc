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

namespace airsched {

constexpr int KR = 4;              // relocate chunk: 4 x 32 target slots cached per lane
constexpr int KS = 2;              // swap chunk: 2 x 32 m2 missions cached per lane
constexpr int MAXTHREADS = 896;    // <= 28 runs per CTA (one wave of 4096 runs on 148 SMs)

struct BatchLayout {
    int T, CS, MH, VC, CH;   // CTA-wide part
    int shared_bytes;
    int RS, LK, BS, F, E;    // per-run part (offsets inside a run block)
    int run_bytes;
};

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline int padded_stride(int NL, int tbytes) {
    if (tbytes == 2) {            // row stride in halfwords = 2 * odd number of words
        int w = (NL + 1) / 2;
        if ((w & 1) == 0) w++;
        return 2 * w;
    }
    return (NL & 1) ? NL : NL + 1; // odd number of words
}

__host__ __device__ inline BatchLayout batch_layout(int n, int V, int NL, int NC, int tbytes, int ebytes, bool tabu) {
    BatchLayout L;
    const int S = n + V;
    const int NLp = padded_stride(NL, tbytes);
    int o = 0;
    L.T = o; o = al16(o + NC * NL * NLp * tbytes);
    L.CS = o; o = al16(o + S * 16);
    L.MH = o; o = al16(o + n);
    L.VC = o; o = al16(o + V * 4);
    L.CH = o; o = al16(o + NC);
    L.shared_bytes = o;
    int r = 0;
    L.RS = r; r = al16(r + S * 16);
    L.LK = r; r = al16(r + S * 4);
    L.BS = r; r = al16(r + S * 2);
    L.F = r; r = al16(r + V * 4);
    L.E = r; r = al16(r + (tabu ? n * V * ebytes : 0));
    L.run_bytes = r;
    return L;
}

void batch_smem(int n, int V, int NL, int NC, int tbytes, int ebytes, bool tabu, size_t *shared_bytes,
                size_t *run_bytes) {
    BatchLayout L = batch_layout(n, V, NL, NC, tbytes, ebytes, tabu);
    *shared_bytes = L.shared_bytes;
    *run_bytes = L.run_bytes;
}

// Mission view over the AoS records (same interface as MissionViewT).
template <class TT>
struct CompactMV {
    const TT *T;
    const unsigned char *CS;
    const uint8_t *MH;
    const uint32_t *VC;
    const uint8_t *CH;
    int32_t n, V, NL, NLp, P, DAY;
    __device__ __forceinline__ int cls(int v) const { return VC[v] & 0xFF; }
    __device__ __forceinline__ int hok(int c) const { return CH[c]; }
    __device__ __forceinline__ int vl(int v) const { return (int)(VC[v] >> 16); }
    __device__ __forceinline__ int dl(int m) const { return *reinterpret_cast<const uint16_t *>(CS + m * 16 + 6); }
    __device__ __forceinline__ int hl(int m) const { return MH[m]; }
    __device__ __forceinline__ int sv(int c, int m) const {
        return *reinterpret_cast<const int32_t *>(CS + m * 16 + 8 + 4 * c);
    }
};

template <class ET>
struct CompactRV {
    Field<uint16_t, 4, 0> succ;
    Field<uint16_t, 4, 2> pred;
    Field<int16_t, 16, 14> veh;
    Field<uint16_t, 16, 12> endc;
    Field<int32_t, 16, 0> depc;
    Field<int32_t, 16, 4> inc;
    Field<int32_t, 16, 8> svco;
    Field<uint16_t, 16, 4> pick_s;
    Field<int32_t, 16, 0> w_s;
    int32_t *F;
    ET *E;
};

__device__ __forceinline__ uint64_t wmin(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t u = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = u < v ? u : v;
    }
    return v;
}

template <class T>
__device__ __forceinline__ T bcast(T v) {
    return __shfl_sync(0xFFFFFFFFu, v, 0);
}

template <bool TABU, class TT, class ET>
__global__ void __launch_bounds__(MAXTHREADS, 1) k_batch(SearchArgs A, int RPC) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DevInst &I = A.inst;
    const int n = I.n, V = I.V, S = n + V, NC = I.NC, NL = I.NL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const BatchLayout L = batch_layout(n, V, NL, NC, (int)sizeof(TT), (int)sizeof(ET), TABU);
    const int NLp = padded_stride(NL, (int)sizeof(TT));
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
    __syncthreads();

    const int run = blockIdx.x * RPC + warp;
    if (warp >= RPC || run >= A.n_runs) return;

    unsigned char *rb = smem + L.shared_bytes + warp * L.run_bytes;
    unsigned char *RSb = rb + L.RS;
    int4 *RS4 = reinterpret_cast<int4 *>(RSb);
    uint32_t *LK = reinterpret_cast<uint32_t *>(rb + L.LK);
    uint16_t *BS = reinterpret_cast<uint16_t *>(rb + L.BS);
    int32_t *F = reinterpret_cast<int32_t *>(rb + L.F);
    ET *E = TABU ? reinterpret_cast<ET *>(rb + L.E) : nullptr;

    CompactMV<TT> M;
    M.T = Ts; M.CS = CS; M.MH = MH; M.VC = VC; M.CH = CH;
    M.n = n; M.V = V; M.NL = NL; M.NLp = NLp; M.P = I.P; M.DAY = I.DAY;
    CompactRV<ET> R;
    R.succ.base = rb + L.LK; R.pred.base = rb + L.LK;
    R.veh.base = RSb; R.endc.base = RSb; R.depc.base = RSb; R.inc.base = RSb; R.svco.base = RSb;
    R.pick_s.base = CS; R.w_s.base = CS;
    R.F = F; R.E = E;

    // ---- start schedule (CSR) -> linked lists --------------------------------
    const int32_t *ptr = A.start_ptr + (A.shared_start ? 0 : (size_t)run * (V + 1));
    const int32_t *ms = A.start_ms + (A.shared_start ? 0 : (size_t)run * n);
    for (int x = lane; x < S; x += 32) R.veh[x] = x < n ? (int16_t)-1 : (int16_t)(x - n);
    if (TABU)
        for (int i = lane; i < n * V; i += 32) E[i] = (ET)-1;
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
        for (int x = lane; x < S; x += 32) {
            if (x < n && R.veh[x] < 0) { bad = 1; continue; }   // unlisted => a duplicate elsewhere
            refresh_slot(M, R, x);
            if (R.depc[x] + R.inc[x] > R.w_s[x]) bad = 1;                          // con7/con8
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
    if (lane == 0) {
        uint64_t seed = A.seeds ? A.seeds[run] : A.seed;
        if (seed != 0 && n > 0) {
            uint64_t s = seed;
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
    const int P = I.P;
    const uint32_t Rb = (uint32_t)n * (uint32_t)S;
    int it = 0, stop = 0;
    for (; it < A.max_iters; it++) {
        __syncwarp();
        uint64_t kmin = KEY_NONE;
        const int asp = (int)(best - cur);   // aspiration: cur + delta < best  <=>  delta < asp

        // Per-lane best inside a block: 32-bit key (class << 31 | delta + 2^30) plus
        // the index.  Each lane visits its items in increasing index order inside a
        // block, so a strict '<' keeps the lowest index among equal keys; blocks are
        // merged through the 64-bit key.
        constexpr int NEG = -(1 << 29);
        const bool en_inter_r = (mask & 1u) != 0, en_intra_r = (mask & 2u) != 0;
        const bool en_inter_s = (mask & 4u) != 0, en_intra_s = (mask & 8u) != 0;

        // ============================ relocate block ============================
        for (int t0 = 0; t0 < S; t0 += 32 * KR) {
            int c_t1[KR], c_t2[KR], c_dw[KR], c_k[KR], c_wsv[KR], c_slk[KR], c_inf[KR];
#pragma unroll
            for (int k = 0; k < KR; k++) {
                const int t = t0 + lane + 32 * k;
                int t1 = 0, t2 = 0, dw = 0, kk = 0, wsv = NEG, slk = NEG, inf = 0xFFFF;
                if (t < S) {
                    const int4 rs = RS4[t];
                    const int b = (int16_t)((uint32_t)rs.w >> 16);
                    if (b >= 0) {
                        const int4 cs = CS4[t];
                        const uint32_t vc = VC[b];
                        const int cb = vc & 0xFF;
                        t1 = (cb * NL + (rs.w & 0xFFFF)) * NLp;     // row of T_cb[endc(t)][.]
                        t2 = cb * NL * NLp + (cs.y & 0xFFFF);        // column pick(t) of T_cb
                        dw = -rs.x;                                  // -dep(pred t)
                        kk = rs.z - rs.y;                            // svco(t) - inc(t)
                        wsv = cs.x - rs.z;                           // w(t) - svco(t)
                        slk = P - F[b];
                        inf = (b & 0xFFFF) | (cb << 16) | (((vc >> 8) & 1) << 20);
                    }
                }
                c_t1[k] = t1; c_t2[k] = t2; c_dw[k] = dw; c_k[k] = kk; c_wsv[k] = wsv; c_slk[k] = slk;
                c_inf[k] = inf;
            }
            uint32_t bk32 = 0xFFFFFFFFu, bidx = 0;
            for (int m = 0; m < n; m++) {
                const int4 rm = RS4[m];
                const int a = (int16_t)((uint32_t)rm.w >> 16);
                if (a < 0) continue;
                const int s = LK[m] & 0xFFFF;
                const int4 rsx = RS4[s];
                const int4 csx = CS4[s];
                const int ca = VC[a] & 0xFF;
                const int Dps = (int)Ts[(ca * NL + (rm.w & 0xFFFF)) * NLp + (csx.y & 0xFFFF)] + rsx.z;
                if (rm.x + Dps > csx.x) continue;     // link p->s infeasible: every relocate of m is
                const int rem = Dps - rm.y - rsx.y;   // removal delta d(p,s) - d(p,m) - d(m,s)
                const int4 cm = CS4[m];
                const int Fa = F[a];
                const int inter_bias = (Fa + rem <= P) ? 0 : NEG;
                const int intra_lim = P - Fa - rem;
                const int w_m = cm.x, pick_m = cm.y & 0xFFFF, rowD = ((uint32_t)cm.y >> 16) * NLp;
                const int svm0 = cm.z, svm1 = cm.w;
                const bool heli_m = MH[m] != 0;
                const ET *Erow = TABU ? E + m * V : nullptr;
                const uint32_t base = (uint32_t)m * (uint32_t)S + t0 + lane;
#pragma unroll
                for (int k = 0; k < KR; k++) {
                    const int t = t0 + lane + 32 * k;
                    const int inf = c_inf[k];
                    const int b = (int)(int16_t)(inf & 0xFFFF);
                    const bool cb1 = (inf >> 16) & 1;
                    const bool hok = (inf >> 20) & 1;
                    const int T1 = (int)Ts[c_t1[k] + pick_m];
                    const int T2 = (int)Ts[c_t2[k] + rowD];
                    const int x1 = T1 + (cb1 ? svm1 : svm0);
                    const int ins = x1 + T2 + c_k[k];
                    const int delta = rem + ins;
                    const bool same = b == a;
                    const int lim = same ? intra_lim : c_slk[k] + inter_bias;
                    const int mg = min(min(w_m + c_dw[k] - x1, c_wsv[k] - w_m - T2), lim - ins);
                    const bool ok = (mg >= 0) & (t != m) & (t != s) & (same ? en_intra_r : en_inter_r) &
                                    (hok | !heli_m);
                    bool adm;
                    if (TABU) adm = ((int)Erow[max(b, 0)] < it) | (delta < asp);
                    else adm = delta < 0;
                    uint32_t k32 = (uint32_t)(delta + DELTA_BIAS) | (adm ? 0u : 0x80000000u);
                    k32 = ok ? k32 : 0xFFFFFFFFu;
                    const bool better = k32 < bk32;
                    bk32 = better ? k32 : bk32;
                    bidx = better ? base + 32 * k : bidx;
                }
            }
            const uint64_t kb = bk32 == 0xFFFFFFFFu ? KEY_NONE : (((uint64_t)bk32 << 32) | bidx);
            kmin = kb < kmin ? kb : kmin;
        }

        // ============================== swap block ==============================
        // m2 chunks of 32*KS aligned to the top (hi = n, n - 64, ...) so only the
        // lowest chunk is ragged; adjacent pairs are excluded here and scored exactly
        // by the generic three-link formula below.
        for (int hi = n; hi > 1; hi -= 32 * KS) {
            const int lo = hi - 32 * KS;
            int q_ps[KS], q_sv0[KS], q_sv1[KS], q_d2[KS], q_e2[KS], q_p2[KS], q_w2[KS], q_dep2[KS], q_kb[KS],
                q_ws2[KS], q_slk[KS], q_inf[KS];
#pragma unroll
            for (int k = 0; k < KS; k++) {
                const int m2 = lo + lane + 32 * k;
                int ps = 0, sv0 = 0, sv1 = 0, d2 = 0, e2 = 0, p2 = 0, w2 = 0, dep2 = 0, kb = 0, ws2 = NEG, slk = NEG,
                    inf = 0xFFFF;
                if (m2 >= 0) {
                    const int4 r2 = RS4[m2];
                    const int b = (int16_t)((uint32_t)r2.w >> 16);
                    if (b >= 0) {
                        const int4 c2 = CS4[m2];
                        const uint32_t vc = VC[b];
                        const int cb = vc & 0xFF;
                        const int s2 = LK[m2] & 0xFFFF;
                        const int4 rs2 = RS4[s2];
                        const int4 cs2 = CS4[s2];
                        ps = (c2.y & 0xFFFF) | (s2 << 16);              // pick2 | s2 << 16
                        sv0 = c2.z;
                        sv1 = c2.w;
                        d2 = ((uint32_t)c2.y >> 16) * NLp;               // row del2 (any class)
                        e2 = (cb * NL + (r2.w & 0xFFFF)) * NLp;           // row T_cb[endc2]
                        p2 = cb * NL * NLp + (cs2.y & 0xFFFF);            // column pick(s2) of T_cb
                        w2 = c2.x;
                        dep2 = r2.x;
                        kb = rs2.z - r2.y - rs2.y;                        // svco(s2) - inc2 - inc(s2)
                        ws2 = cs2.x - rs2.z;                              // w(s2) - svco(s2)
                        slk = P - F[b];
                        inf = (b & 0xFFFF) | (cb << 16) | ((int)MH[m2] << 20) | (((vc >> 8) & 1) << 21);
                    }
                }
                q_ps[k] = ps; q_sv0[k] = sv0; q_sv1[k] = sv1; q_d2[k] = d2; q_e2[k] = e2; q_p2[k] = p2;
                q_w2[k] = w2; q_dep2[k] = dep2; q_kb[k] = kb; q_ws2[k] = ws2; q_slk[k] = slk; q_inf[k] = inf;
            }
            uint32_t bk32 = 0xFFFFFFFFu, bidx = 0;
            for (int m1 = 0; m1 <= hi - 2; m1++) {
                const int4 r1 = RS4[m1];
                const int a = (int16_t)((uint32_t)r1.w >> 16);
                if (a < 0) continue;
                const int s1 = LK[m1] & 0xFFFF;
                const int4 c1 = CS4[m1];
                const int4 rs1 = RS4[s1];
                const int4 cs1 = CS4[s1];
                const uint32_t vca = VC[a];
                const int ca = vca & 0xFF;
                const bool hoka = (vca >> 8) & 1;
                const int row_ya1 = (ca * NL + (r1.w & 0xFFFF)) * NLp;  // T_ca[endc1][.]
                const int col_ta2 = ca * NL * NLp + (cs1.y & 0xFFFF);    // T_ca[.][pick(s1)]
                const int pick1 = c1.y & 0xFFFF, row_tb2 = ((uint32_t)c1.y >> 16) * NLp;
                const int depc1 = r1.x, w1 = c1.x;
                const bool heli1 = MH[m1] != 0;
                const int wsv1 = cs1.x - rs1.z;                 // w(s1) - svco(s1)
                const int ka = rs1.z - r1.y - rs1.y;            // svco(s1) - inc1 - inc(s1)
                const int slkA = P - F[a];
                const int sv10 = c1.z, sv11 = c1.w;
                const ET *Erow = TABU ? E + m1 * V : nullptr;
                const uint32_t base = Rb + (uint32_t)m1 * (uint32_t)n + lo + lane;
#pragma unroll
                for (int k = 0; k < KS; k++) {
                    if (lo + 32 * k + 31 <= m1) continue;     // sub-chunk entirely on or below the diagonal
                    const int m2 = lo + lane + 32 * k;
                    const int inf = q_inf[k];
                    const int b = (int)(int16_t)(inf & 0xFFFF);
                    const bool cb1 = (inf >> 16) & 1;
                    const bool h2 = (inf >> 20) & 1, hokb = (inf >> 21) & 1;
                    const int pick2 = q_ps[k] & 0xFFFF, s2 = (uint32_t)q_ps[k] >> 16;
                    const bool same = a == b;
                    const int ya1 = (int)Ts[row_ya1 + pick2] + (ca ? q_sv1[k] : q_sv0[k]);   // p1 -> m2
                    const int Ta2 = (int)Ts[col_ta2 + q_d2[k]];                              // m2 -> s1
                    const int yb1 = (int)Ts[q_e2[k] + pick1] + (cb1 ? sv11 : sv10);          // p2 -> m1
                    const int Tb2 = (int)Ts[q_p2[k] + row_tb2];                              // m1 -> s2
                    const int da = ya1 + Ta2 + ka;
                    const int db = yb1 + Tb2 + q_kb[k];
                    const int delta = da + db;
                    const int mf = same ? slkA - delta : min(slkA - da, q_slk[k] - db);
                    const int mg = min(min(min(q_w2[k] - depc1 - ya1, wsv1 - q_w2[k] - Ta2),
                                           min(w1 - q_dep2[k] - yb1, q_ws2[k] - w1 - Tb2)), mf);
                    const bool ok = (mg >= 0) & (m2 > m1) & (s1 != m2) & (s2 != m1) &
                                    (same ? en_intra_s : en_inter_s) & (!h2 | hoka) & (!heli1 | hokb);
                    bool adm;
                    if (TABU) adm = (((int)Erow[max(b, 0)] < it) & ((int)E[max(m2, 0) * V + a] < it)) | (delta < asp);
                    else adm = delta < 0;
                    uint32_t k32 = (uint32_t)(delta + DELTA_BIAS) | (adm ? 0u : 0x80000000u);
                    k32 = ok ? k32 : 0xFFFFFFFFu;
                    const bool better = k32 < bk32;
                    bk32 = better ? k32 : bk32;
                    bidx = better ? base + 32 * k : bidx;
                }
            }
            const uint64_t kb = bk32 == 0xFFFFFFFFu ? KEY_NONE : (((uint64_t)bk32 << 32) | bidx);
            kmin = kb < kmin ? kb : kmin;
        }
        // adjacent pairs (x, succ x): the exact three-link formula (engine.cuh)
        if (mask & 8u) {
            for (int x = lane; x < n; x += 32) {
                const int g = LK[x] & 0xFFFF;
                if (R.veh[x] < 0 || g >= n) continue;
                const int m1 = min(x, g), m2 = max(x, g);
                const MoveEval e = swap_eval(M, R, m1, m2, mask, it);
                const int cls = move_class<TABU>(e, cur, best);
                if (cls >= 0) {
                    const uint64_t key = make_key(cls, e.delta, Rb + (uint32_t)m1 * (uint32_t)n + (uint32_t)m2);
                    kmin = key < kmin ? key : kmin;
                }
            }
        }

        // ============================ select + apply ============================
        kmin = wmin(kmin);
        int improved = 0;
        if (lane == 0) {
            if (kmin == KEY_NONE) stop = AS_STOP_NO_MOVE;
            else if (key_cls(kmin) == 1 && (!TABU || A.strict_tabu_stop)) stop = TABU ? AS_STOP_NO_MOVE : AS_STOP_LOCAL_OPT;
            if (!stop) {
                const uint32_t idx = key_idx(kmin);
                MoveEval e = eval_index(M, R, idx, mask, it);
                apply_move(M, R, idx, e, it, A.tenure, TABU);
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

template <bool TABU, class TT, class ET>
static cudaError_t launch_one(const SearchArgs &A, int RPC, size_t smem, cudaStream_t st) {
    cudaError_t err = cudaFuncSetAttribute(k_batch<TABU, TT, ET>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int grid = (A.n_runs + RPC - 1) / RPC;
    k_batch<TABU, TT, ET><<<grid, RPC * 32, smem, st>>>(A, RPC);
    return cudaGetLastError();
}

cudaError_t launch_batch(const SearchArgs &A, int mode, int RPC, int tbytes, int ebytes, size_t smem,
                         cudaStream_t st) {
    if (mode == 1) {
        if (tbytes == 2) return ebytes == 2 ? launch_one<true, uint16_t, int16_t>(A, RPC, smem, st)
                                            : launch_one<true, uint16_t, int32_t>(A, RPC, smem, st);
        return ebytes == 2 ? launch_one<true, int32_t, int16_t>(A, RPC, smem, st)
                           : launch_one<true, int32_t, int32_t>(A, RPC, smem, st);
    }
    if (tbytes == 2) return launch_one<false, uint16_t, int16_t>(A, RPC, smem, st);
    return launch_one<false, int32_t, int16_t>(A, RPC, smem, st);
}

}  // namespace airsched
