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

// Rare path: an adjacent swap whose two deadlines are equal (the only case in
// which it can be feasible on a feasible state), via engine code.
template <class MV, class RV>
__device__ __noinline__ MoveEval adjacent_swap(const MV &M, const RV &R, int m1, int m2, uint32_t mask, int it) {
    return swap_eval(M, R, m1, m2, mask, it);
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

        // ============================ relocate block ============================
        for (int t0 = 0; t0 < S; t0 += 32 * KR) {
            int c_info[KR], c_loc[KR], c_dep[KR], c_k[KR], c_wsv[KR], c_slk[KR];
#pragma unroll
            for (int k = 0; k < KR; k++) {
                const int t = t0 + lane + 32 * k;
                int info = 0xFFFF, loc = 0, dp = 0, kk = 0, wsv = 0, slk = 0;
                if (t < S) {
                    const int4 rs = RS4[t];
                    const int b = (int16_t)((uint32_t)rs.w >> 16);
                    if (b >= 0) {
                        const int4 cs = CS4[t];
                        const uint32_t vc = VC[b];
                        info = (b & 0xFFFF) | ((vc & 0xFF) << 16) | (((vc >> 8) & 1) << 20);
                        loc = (rs.w & 0xFFFF) | (cs.y << 16);     // endc | pick << 16
                        dp = rs.x;
                        kk = rs.z - rs.y;                          // svco - inc
                        wsv = cs.x - rs.z;                         // w - svco
                        slk = P - F[b];
                    }
                }
                c_info[k] = info;
                c_loc[k] = loc;
                c_dep[k] = dp;
                c_k[k] = kk;
                c_wsv[k] = wsv;
                c_slk[k] = slk;
            }
            for (int m = 0; m < n; m++) {
                const int4 rm = RS4[m];
                const int a = (int16_t)((uint32_t)rm.w >> 16);
                if (a < 0) continue;
                const int s = LK[m] & 0xFFFF;
                const int4 cm = CS4[m];
                const int4 rsx = RS4[s];
                const int w_s = *reinterpret_cast<const int32_t *>(CS + s * 16);
                const int pick_s = *reinterpret_cast<const uint16_t *>(CS + s * 16 + 4);
                const int ca = VC[a] & 0xFF;
                const int Dps = (int)Ts[(ca * NL + (rm.w & 0xFFFF)) * NLp + pick_s] + rsx.z;
                const int rem = Dps - rm.y - rsx.y;
                const bool rem_ok = rm.x + Dps <= w_s;
                const int Fa = F[a];
                const bool inter_ok = rem_ok && (Fa + rem <= P);
                const int intra_lim = P - Fa - rem;
                const int w_m = cm.x, pick_m = cm.y & 0xFFFF, del_m = (uint32_t)cm.y >> 16;
                const int svm0 = cm.z, svm1 = cm.w;
                const bool heli_m = MH[m] != 0;
                const ET *Erow = TABU ? E + m * V : nullptr;
                const uint32_t base = (uint32_t)m * (uint32_t)S;
#pragma unroll
                for (int k = 0; k < KR; k++) {
                    const int t = t0 + lane + 32 * k;
                    const int info = c_info[k];
                    const int b = (int)(int16_t)(info & 0xFFFF);
                    const int cb = (info >> 16) & 0xF;
                    const bool hok = (info >> 20) & 1;
                    const bool same = b == a;
                    // branch-free: every lane evaluates, invalid lanes are masked out of the key
                    bool ok = (b >= 0) & (t != m) & (t != s) & ((mask & (same ? 2u : 1u)) != 0);
                    const int e = c_loc[k] & 0xFFFF, pk = (uint32_t)c_loc[k] >> 16;
                    const int T1 = (int)Ts[(cb * NL + e) * NLp + pick_m];
                    const int T2 = (int)Ts[(cb * NL + del_m) * NLp + pk];
                    const int x1 = T1 + (cb ? svm1 : svm0);
                    const int ins = x1 + T2 + c_k[k];
                    const int delta = rem + ins;
                    ok = ok & (hok | !heli_m) & (x1 <= w_m - c_dep[k]) & (T2 <= c_wsv[k] - w_m);
                    ok = ok & (same ? (rem_ok & (ins <= intra_lim)) : (inter_ok & (ins <= c_slk[k])));
                    bool adm;
                    if (TABU) {
                        const bool tabu = (int)Erow[max(b, 0)] >= it;
                        adm = !tabu | (delta < asp);
                    } else {
                        adm = delta < 0;
                    }
                    const uint64_t key = make_key(adm ? 0 : 1, delta, base + (uint32_t)t);
                    kmin = (ok && key < kmin) ? key : kmin;
                }
            }
        }

        // ============================== swap block ==============================
        for (int c0 = 0; c0 < n; c0 += 32 * KS) {
            int q_info[KS], q_loc[KS], q_dls[KS], q_s2[KS], q_dep[KS], q_w[KS], q_kb[KS], q_ws2[KS], q_slk[KS];
            int q_svc0[KS], q_svc1[KS];
#pragma unroll
            for (int k = 0; k < KS; k++) {
                const int m2 = c0 + lane + 32 * k;
                int info = 0xFFFF, loc = 0, dls = 0, s2 = 0, dp = 0, w2 = 0, kb = 0, ws2 = 0, slk = 0, sv0 = 0, sv1 = 0;
                if (m2 < n) {
                    const int4 r2 = RS4[m2];
                    const int b = (int16_t)((uint32_t)r2.w >> 16);
                    if (b >= 0) {
                        const int4 c2 = CS4[m2];
                        const uint32_t vc = VC[b];
                        s2 = LK[m2] & 0xFFFF;
                        const int4 rs2 = RS4[s2];
                        const int w_s2 = *reinterpret_cast<const int32_t *>(CS + s2 * 16);
                        const int pick_s2 = *reinterpret_cast<const uint16_t *>(CS + s2 * 16 + 4);
                        info = (b & 0xFFFF) | ((vc & 0xFF) << 16) | ((int)MH[m2] << 20) | (((vc >> 8) & 1) << 21);
                        loc = (r2.w & 0xFFFF) | ((c2.y & 0xFFFF) << 16);           // endc2 | pick2 << 16
                        dls = ((uint32_t)c2.y >> 16) | (pick_s2 << 16);            // del2 | pick(s2) << 16
                        dp = r2.x;
                        w2 = c2.x;
                        kb = rs2.z - r2.y - rs2.y;                                 // svco(s2) - inc2 - inc(s2)
                        ws2 = w_s2 - rs2.z;                                        // w(s2) - svco(s2)
                        slk = P - F[b];
                        sv0 = c2.z;
                        sv1 = c2.w;
                    }
                }
                q_info[k] = info;
                q_loc[k] = loc;
                q_dls[k] = dls;
                q_s2[k] = s2;
                q_dep[k] = dp;
                q_w[k] = w2;
                q_kb[k] = kb;
                q_ws2[k] = ws2;
                q_slk[k] = slk;
                q_svc0[k] = sv0;
                q_svc1[k] = sv1;
            }
            const int last_row = min(n - 2, c0 + 32 * KS - 2);
            for (int m1 = 0; m1 <= last_row; m1++) {
                const int4 r1 = RS4[m1];
                const int a = (int16_t)((uint32_t)r1.w >> 16);
                if (a < 0) continue;
                const int s1 = LK[m1] & 0xFFFF;
                const int4 c1 = CS4[m1];
                const int4 rs1 = RS4[s1];
                const int w_s1 = *reinterpret_cast<const int32_t *>(CS + s1 * 16);
                const int pick_s1 = *reinterpret_cast<const uint16_t *>(CS + s1 * 16 + 4);
                const uint32_t vca = VC[a];
                const int ca = vca & 0xFF;
                const bool hoka = (vca >> 8) & 1;
                const int endc1 = r1.w & 0xFFFF, depc1 = r1.x;
                const int pick1 = c1.y & 0xFFFF, del1 = (uint32_t)c1.y >> 16, w1 = c1.x;
                const bool heli1 = MH[m1] != 0;
                const int wsv1 = w_s1 - rs1.z;                 // w(s1) - svco(s1)
                const int ka = rs1.z - r1.y - rs1.y;           // svco(s1) - inc1 - inc(s1)
                const int slkA = P - F[a];
                const int sv10 = c1.z, sv11 = c1.w;
                const ET *Erow = TABU ? E + m1 * V : nullptr;
                const uint32_t base = Rb + (uint32_t)m1 * (uint32_t)n;
#pragma unroll
                for (int k = 0; k < KS; k++) {
                    if (c0 + 32 * k + 31 <= m1) continue;     // whole sub-chunk on or below the diagonal
                    const int m2 = c0 + lane + 32 * k;
                    const int info = q_info[k];
                    const int b = (int)(int16_t)(info & 0xFFFF);
                    const int cb = (info >> 16) & 0xF;
                    const bool h2 = (info >> 20) & 1, hokb = (info >> 21) & 1;
                    const bool same = a == b;
                    bool ok = (m2 > m1) & (b >= 0) & ((mask & (same ? 8u : 4u)) != 0);
                    const bool adj = (s1 == m2) || (q_s2[k] == m1);
                    const int e2 = q_loc[k] & 0xFFFF, p2 = (uint32_t)q_loc[k] >> 16;
                    const int d2 = q_dls[k] & 0xFFFF, ps2 = (uint32_t)q_dls[k] >> 16;
                    const int ya1 = (int)Ts[(ca * NL + endc1) * NLp + p2] + (ca ? q_svc1[k] : q_svc0[k]); // p1 -> m2
                    const int Ta2 = (int)Ts[(ca * NL + d2) * NLp + pick_s1];                           // m2 -> s1
                    const int yb1 = (int)Ts[(cb * NL + e2) * NLp + pick1] + (cb ? sv11 : sv10);        // p2 -> m1
                    const int Tb2 = (int)Ts[(cb * NL + del1) * NLp + ps2];                             // m1 -> s2
                    const int da = ya1 + Ta2 + ka;
                    const int db = yb1 + Tb2 + q_kb[k];
                    int delta = da + db;
                    bool f = (!h2 | hoka) & (!heli1 | hokb) & (depc1 + ya1 <= q_w[k]) & (q_w[k] + Ta2 <= wsv1) &
                             (q_dep[k] + yb1 <= w1) & (Tb2 <= q_ws2[k] - w1);
                    f = f & (same ? (delta <= slkA) : ((da <= slkA) & (db <= q_slk[k])));
                    if (adj) {
                        // adjacent pair: feasible only if both deadlines are equal;
                        // then take the exact three-link formula.
                        f = false;
                        if (ok && q_w[k] == w1) {
                            MoveEval ev = adjacent_swap(M, R, m1, m2, mask, it);
                            f = ev.feasible;
                            delta = ev.delta;
                        }
                    }
                    ok = ok & f;
                    bool adm;
                    if (TABU) {
                        const int m2c = m2 < n ? m2 : 0;
                        const bool tabu = ((int)Erow[max(b, 0)] >= it) | ((int)E[m2c * V + a] >= it);
                        adm = !tabu | (delta < asp);
                    } else {
                        adm = delta < 0;
                    }
                    const uint64_t key = make_key(adm ? 0 : 1, delta, base + (uint32_t)m2);
                    kmin = (ok && key < kmin) ? key : kmin;
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
