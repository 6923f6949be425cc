// window.cuh -- the WINDOW scorers of the batched kernel (k_batch, one run per
// warp): the same moves, formulas and keys as score.cuh's FAST scorers, with
// the warp-uniform per-row work taken out of the scoring loops.
//
// In a tile every lane scores the same row m (m1) against its own targets, so
// everything that depends only on the row is the same for all 32 lanes.  The
// FAST scorers recompute it per row in every lane (~60 SASS instructions per
// row, and the register pressure of 28 warps x 72 registers makes the compiler
// rematerialise part of it inside the item loop).  Here the rows are taken 32
// at a time: lane j builds row (w0 + j)'s record once (lane-parallel), stores it
// in the warp's window buffer, and the row loop reads it back with broadcast
// LDS.128s.  Four more changes cut the per-move instruction count:
//
//  * tabu test by bitmask: TB[m] bit (31 - v) is set iff E[m][v] >= it (O8), so
//    "placed-into pair (m, b) is tabu" is the sign bit of TB[m] << b -- one shift
//    instead of a gather of the expiry matrix (which moves to global memory:
//    the scorers never read it; apply writes it; V <= 32);
//  * node costs staged per CTA: TD_c[x][m] = d_c(x, m) = T_c[x][pick_m] +
//    T_c[pick_m][del_m] (O2, uint16; the host checks the largest fits), so
//    the cost of arriving at a mission is one gather instead of a gather, the
//    service leg of the right class and two adds; the swap's d_a(p1, m2) reads
//    one TD row over consecutive lanes (no bank conflicts), and the gathers
//    whose lanes vary the origin x read the transposed copy TDT_c[m][x] (one
//    row per class instead of a column);
//  * row-local table read where a gather would read down a column: the swap's
//    T_ca[del m2][pick s1] is read from the per-layer transpose (T itself when
//    every layer is symmetric, else a transposed copy staged next to T);
//  * sums as 3-input adds (IADD3, ALU pipe) or mad.lo (FMA pipe), split so
//    neither half-rate pipe limits the issue rate;
//  * per-lane 32-bit key with a local index: bit 31 = not admissible, bits
//    7..30 = delta + 2^23, bits 0..6 = the lane's item number inside the window
//    (row * KR + k or row * KS + k, increasing with the canonical index), so
//    the running best is one unsigned min; the window's winner is turned into
//    the 64-bit (class, delta, index) key at the window's end.  Needs |delta| <
//    2^23: true for uint16 tables (|delta| < 8 * 2^16);
//  * feasibility margins combined by OR (the sign of a | b | c is set iff one
//    of them is negative) and the infeasible poison by an arithmetic shift;
//  * no same-route branch (reading #42): with every pickup->delivery
//    leg > 0 (svcpos, required by the FAST scorers) a feasible route is strictly
//    deadline-sorted, so every intra-route relocate or swap fails
//    one of its new-link checks; the flight-limit margins therefore use the
//    inter-route form for every move, and a row whose removal leaves route a
//    over the flight limit (F_a + rem > P) has no feasible move at all and is
//    skipped.  Results are identical; the parity suite checks traces bit-exact.
#pragma once
#include <cstdint>
#include <type_traits>

#include "score.cuh"

namespace airsched {

constexpr int WIN_ROWS = 32;                 // rows per window (one per lane)
constexpr int WIN_REC_INT4 = 3;              // record size (int4 words) of the larger (swap) record
constexpr int WIN_KEY_SHIFT = 7;             // local-index bits of the 32-bit key
constexpr int WIN_BIAS = 1 << 23;            // delta bias of the 32-bit key
constexpr uint32_t WIN_NONE = 0xFFFFFFFFu;
constexpr int WIN_HELI_OFF = 1 << 30;        // lane slack offset: vehicle may not fly a heli-only mission

struct WinCtx {
    int4 *WB;               // [WIN_ROWS][WIN_REC_INT4] this warp's window buffer (shared)
    const uint32_t *TB;     // [n] tabu bits: bit (31 - v) of TB[m] <=> E[m][v] >= it (TABU only)
    int ttsm;               // shared-window byte address of the transposed table (== the table's when symmetric)
    int tdsm;               // shared-window byte address of TD[NC][LTD] (uint16 node costs d_c(x, t), rows NTDp)
    int tdtsm;              // ... of TDT[NC][n][NLp] (the same, transposed per class)
    int NTDp, LTD;          // TD row stride and class-layer stride (halfwords, compact.cuh td_layer)
};

// x * p on the FMA pipe (IMAD); with p = 2^s it is x << s.  The tabu-bit shifts are written this way so they
// leave the ALU pipe, the busier of the two (ncu: ALU 73 %, FMA 30 % of their peaks in k_batch).
__device__ __forceinline__ uint32_t mul_fma(uint32_t x, uint32_t p) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(x), "r"(p));
    return r;
}

__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t s) {   // x << s, 0 when s >= 32 (PTX shl)
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
}

// ld.shared.u16 at a 32-bit shared-window byte address plus an immediate offset (folded into the LDS)
template <int OFF>
__device__ __forceinline__ int lds_u16_off(uint32_t addr) {
    unsigned short v;
    asm("ld.shared.u16 %0, [%1+%2];" : "=h"(v) : "r"(addr), "n"(OFF));
    return (int)v;
}

// 32-bit window key -> 64-bit key (class << 63 | (delta + 2^30) << 32 | idx)
__device__ __forceinline__ uint64_t win_key64(uint32_t bk, uint32_t idx) {
    const uint32_t d = ((bk >> WIN_KEY_SHIFT) & 0xFFFFFFu) + (uint32_t)(DELTA_BIAS - WIN_BIAS);
    return ((uint64_t)((bk & 0x80000000u) | d) << 32) | idx;
}

// ---------------------------------------------------------------------------
// Relocate block: move m (route a, p -> m -> s) to just before slot t (route b, c -> t).
// Record of row m (2 int4):
//   q0 = {remk, hmask, w_m, rowD}   remk = (rem + 2^23) << 7 | r * KR (key base; item k adds k);
//        hmask = 0x3FFFFFFF (m not heli-only) or ~0 (heli-only); w_m = NEG for a row without a feasible
//        move; rowD = byte offset of TD row del_m
//   q1 = {TB[m], rem - asp (TS) or rem (NS), byte offset of TDT row m, 0}
template <bool TABU, bool SV>
__device__ __forceinline__ void win_reloc_record(const ScoreCtx<uint16_t, int32_t> &C, const WinCtx &W, int m, int r,
                                                 int asp) {
    // a row without a feasible move keeps w_m = NEG: its first link margin is negative for every target,
    // so the row loop needs no skip test (such rows are rare: by the triangle inequality the removal
    // link p -> s and route a's total after the removal are normally feasible)
    int4 q0 = make_int4(0, 0x3FFFFFFF, NEG, 0), q1 = make_int4(0, 0, 0, 0), q2 = make_int4(0, 0, 0, 0);
    const int4 rm = C.RS4[m];
    const int a = (int16_t)((uint32_t)rm.w >> 16);
    if (a >= 0) {
        const int s = C.LK[m] & 0xFFFF;
        const int4 rsx = C.RS4[s];
        const int4 csx = C.CS4[s];
        const int ca = C.VC[a] & 0xFF;
        const int Dps = (int)C.Ts[(ca * C.NL + (rm.w & 0xFFFF)) * C.NLp + (csx.y & 0xFFFF)] + rsx.z;
        const int rem = Dps - rm.y - rsx.y;   // removal delta d(p,s) - d(p,m) - d(m,s)
        // link p->s (con7/con8); with positive legs (SV) also route a's flight total after the removal
        // (con6, reading #42: no intra-route move is feasible, so no move of the row is)
        if (rm.x + Dps <= csx.x && (!SV || C.F[a] + rem <= C.P)) {
            const int4 cm = C.CS4[m];
            q0 = make_int4((rem + WIN_BIAS) * (1 << WIN_KEY_SHIFT) + r * KR, C.MH[m] ? (int)0xFFFFFFFF : 0x3FFFFFFF,
                           cm.x, 2 * (int)((uint32_t)cm.y >> 16) * W.NTDp);
            q1 = make_int4(TABU ? (int)W.TB[m] : 0, TABU ? rem - asp : rem, 2 * m * C.NLp, s);
            // general legs: the same-route limit P - F_a - rem, and the inter-route bias (NEG when the
            // removal alone leaves route a over the limit)
            q2 = make_int4(C.P - C.F[a] - rem, C.F[a] + rem <= C.P ? 0 : NEG, a, 0);
        }
    }
    int4 *rec = W.WB + r * WIN_REC_INT4;
    rec[0] = q0; rec[1] = q1;
    if (!SV) rec[2] = q2;
}

// F1 (positive legs only): one sign bit for "not admissible OR infeasible" -- k32 = key | ((nadm | margins) & 2^31),
// one ALU instruction fewer per move than the exact form (nadm << 31 | key, all ones when infeasible).  A window
// minimum below 2^31 is then exactly the exact form's (the same admissible feasible moves, the same order); a
// minimum at or above 2^31 says only that no admissible feasible move exists, and the caller re-scores the
// iteration with the exact form (batch.cu) -- rare in TS, once per NS run.
template <bool TABU, bool SV, bool F1 = false>
__device__ __forceinline__ uint64_t score_reloc_win(const ScoreCtx<uint16_t, int32_t> &C, const WinCtx &W, int t0,
                                                    int m_lo, int m_hi, int it, int asp, int lane) {
    const int4 *CS4 = C.CS4, *RS4 = C.RS4;
    const uint32_t *VC = C.VC;
    const int S = C.S, NL = C.NL, NLp = C.NLp, P = C.P;
    const int one = C.one, neg = C.neg;
    const int tsm = (int)__cvta_generic_to_shared(C.Ts);
    // target-slot side, per lane; c_slk carries the heli offset
    int c_x1[KR], c_t2[KR], c_dw[KR], c_k[KR], c_wsv[KR], c_slk[KR], c_b[KR];
    uint32_t c_p2[KR];   // 2^b (0 for a lane without a target): the tabu-bit shift as a multiplication
#pragma unroll
    for (int k = 0; k < KR; k++) {
        const int t = t0 + lane + 32 * k;
        int x1 = W.tdtsm, t2 = W.tdsm, dw = 0, kk = 0, wsv = NEG, slk = 0, b = 0xFFFF;
        if (t < S) {
            const int4 rs = RS4[t];
            const int bb = (int16_t)((uint32_t)rs.w >> 16);
            if (bb >= 0) {
                const int4 cs = CS4[t];
                const uint32_t vc = VC[bb];
                const int cb = vc & 0xFF;
                b = bb;
                x1 = W.tdtsm + 2 * (cb * C.n * NLp + (rs.w & 0xFFFF));      // TDT_cb column endc(t) (row m)
                t2 = W.tdsm + 2 * (cb * W.LTD + t);                          // TD_cb column t (row del_m)
                dw = -rs.x;                                                 // -dep(pred t)
                kk = -rs.y;                                                 // -inc(t)
                wsv = cs.x;                                                 // w(t)
                slk = (P - C.F[bb]) - (((vc >> 8) & 1) ? 0 : WIN_HELI_OFF);
            }
        }
        c_x1[k] = x1; c_t2[k] = t2; c_dw[k] = dw; c_k[k] = kk; c_wsv[k] = wsv; c_slk[k] = slk; c_b[k] = b;
        c_p2[k] = b < 32 ? 1u << b : 0u;
    }
    uint64_t best = KEY_NONE;
    for (int w0 = m_lo; w0 < m_hi; w0 += WIN_ROWS) {
        __syncwarp();
        if (w0 + lane < m_hi) win_reloc_record<TABU, SV>(C, W, w0 + lane, lane, asp);
        __syncwarp();
        const int nr = min(WIN_ROWS, m_hi - w0);
        uint32_t bk = WIN_NONE;
        for (int r = 0; r < nr; r++) {
            const int4 *rec = W.WB + r * WIN_REC_INT4;
            const int4 q0 = rec[0];
            const int hmask = q0.y;
            const int4 q1 = rec[1];
            const int remk = q0.x, w_m = q0.z, rowD = q0.w;
            const uint32_t tb = (uint32_t)q1.x;
            const int remasp = q1.y, rowM = q1.z, sm = q1.w;
            int intra_lim = 0, inter_bias = 0, am = 0;
            if (!SV) {
                const int4 q2 = rec[2];
                intra_lim = q2.x; inter_bias = q2.y; am = q2.z;
            }
            const int m = w0 + r;
#pragma unroll
            for (int k = 0; k < KR; k++) {
                const int x1 = lds_t<uint16_t>((uint32_t)madd(c_x1[k], one, rowM));    // d_cb(c, m)
                const int T2 = lds_t<uint16_t>((uint32_t)madd(c_t2[k], one, rowD));    // d_cb(m, t)
                const int ins = x1 + T2 + c_k[k];                                       // insertion delta
                const int mA = madd(x1, neg, madd(w_m, one, c_dw[k]));                 // dep(c) + d(c,m) <= w_m
                const int mB = c_wsv[k] - w_m - T2;                                     // w_m + d(m,t) <= w(t)
                int mg;
                if (SV) {
                    const int mC = madd(ins, neg, c_slk[k] & hmask);                    // F_b + ins <= P (+ heli)
                    mg = mA | mB | mC;
                } else {   // general legs: same-route flight limit, explicit no-op targets (t = m, t = succ m)
                    const int t = t0 + lane + 32 * k;
                    const int lim = c_b[k] == am ? intra_lim : (c_slk[k] & hmask) + inter_bias;
                    const int noop = (t == m) | (t == sm) ? -1 : 0;
                    mg = mA | mB | (lim - ins) | noop;
                }
                const int e2 = madd(ins, one, remasp);                                  // delta - asp (TS) / delta (NS)
                uint32_t k32;
                if (F1 && SV) {
                    const uint32_t nz = TABU ? mul_fma(tb, c_p2[k]) & ~(uint32_t)e2 : ~(uint32_t)e2;
                    k32 = (uint32_t)madd(ins, 1 << WIN_KEY_SHIFT, remk + k) | ((nz | (uint32_t)mg) & 0x80000000u);
                } else {
                    uint32_t nadm;
                    if (TABU) nadm = mul_fma(tb, c_p2[k]) & ~(uint32_t)e2 & 0x80000000u;
                    else nadm = ~(uint32_t)e2 & 0x80000000u;
                    k32 = (uint32_t)madd(ins, 1 << WIN_KEY_SHIFT, remk + k) | nadm | (uint32_t)(mg >> 31);
                }
                bk = min(bk, k32);
            }
        }
        if (bk != WIN_NONE) {
            const int lid = bk & ((1 << WIN_KEY_SHIFT) - 1);
            const uint32_t idx = (uint32_t)(w0 + lid / KR) * (uint32_t)S + (uint32_t)(t0 + lane + 32 * (lid % KR));
            const uint64_t key = win_key64(bk, idx);
            best = key < best ? key : best;
        }
    }
    return best;
}

// ---------------------------------------------------------------------------
// Swap block: exchange m1 (route a, p1 -> m1 -> s1) and m2 (route b, p2 -> m2 -> s2), non-adjacent,
// m1 < m2; m2 over the lanes in a top-aligned chunk of 32 * KS (as score_swap_fast).
// Record of row m1 (3 int4); TS folds the aspiration threshold asp into ka, slkA and keyb, so the
// scorer's "delta" is delta - asp (its sign is the aspiration test) and the key still encodes delta:
//   q0 = {cmask | s1 << 8 | a, TD_ca row endc1, Tt_ca row pick(s1), T row del1}   (byte addresses /
//        offsets); cmask = bit 31 when route a cannot fly heli-only missions
//   q1 = {-depc1, w1, w(s1) - svco(s1), svco(s1) - inc1 - inc(s1) - asp}
//   q2 = {P - F_a - asp, keyb = (2^23 + asp) << 7 | r * KS, TB[m1], hmask}
template <bool TABU, bool SV>
__device__ __forceinline__ void win_swap_record(const ScoreCtx<uint16_t, int32_t> &C, const WinCtx &W, int m1, int r,
                                                int tsm, int asp) {
    // an unassigned m1 (partial schedules) keeps -depc1 = NEG: every move of the row fails its first
    // link margin, so the row loop needs no skip test; the table offsets stay valid addresses
    int4 q0 = make_int4(0, W.tdsm, W.ttsm, 0), q1 = make_int4(NEG, 0, 0, 0), q2 = make_int4(0, 0, 0, 0x3FFFFFFF);
    const int4 r1 = C.RS4[m1];
    const int a = (int16_t)((uint32_t)r1.w >> 16);
    if (a >= 0) {
        const int s1 = C.LK[m1] & 0xFFFF;
        const int4 c1 = C.CS4[m1];
        const int4 rs1 = C.RS4[s1];
        const int4 cs1 = C.CS4[s1];
        const uint32_t vca = C.VC[a];
        const int ca = vca & 0xFF;
        const int sa = TABU ? asp : 0;
        q0 = make_int4((((vca >> 8) & 1) ? 0 : (int)0x80000000) | a | (s1 << 8),
                       W.tdsm + 2 * (ca * W.LTD + (r1.w & 0xFFFF) * W.NTDp),       // TD_ca[endc1][.]
                       W.ttsm + 2 * ((ca * C.NL + (cs1.y & 0xFFFF)) * C.NLp),       // Tt_ca[pick(s1)][.]
                       2 * (int)((uint32_t)c1.y >> 16) * C.NLp);                    // T_.[del1][.]
        q1 = make_int4(-r1.x, c1.x, cs1.x - rs1.z, rs1.z - r1.y - rs1.y - sa);
        q2 = make_int4(C.P - C.F[a] - sa, (WIN_BIAS + sa) * (1 << WIN_KEY_SHIFT) + r * KS,
                       TABU ? (int)W.TB[m1] : 0, C.MH[m1] ? (int)0xFFFFFFFF : 0x3FFFFFFF);
    }
    int4 *rec = W.WB + r * WIN_REC_INT4;
    rec[0] = q0; rec[1] = q1; rec[2] = q2;
}

template <bool TABU, bool SV, bool F1 = false>
__device__ __forceinline__ uint64_t score_swap_win(const ScoreCtx<uint16_t, int32_t> &C, const WinCtx &W, int hi,
                                                   int m1_lo, int m1_hi, int it, int asp, int lane) {
    const int4 *CS4 = C.CS4, *RS4 = C.RS4;
    const uint8_t *MH = C.MH;
    const uint32_t *VC = C.VC, *LK = C.LK;
    const int n = C.n, NL = C.NL, NLp = C.NLp, P = C.P;
    const uint32_t Rb = C.Rb;
    const int one = C.one, neg = C.neg;
    const int lo = hi - 32 * KS;
    const int tsm = (int)__cvta_generic_to_shared(C.Ts);
    // m2 side, per lane; q_bf = b | heli_only(m2) << 31, q_slk carries the heli offset
    int q_d2[KS], q_e2[KS], q_p2[KS], q_w2[KS], q_dep2[KS], q_kb[KS], q_ws2[KS], q_slk[KS], q_bf[KS];
    int q_s2[KS];   // general legs only: succ(m2), for the adjacent pairs
    uint32_t q_tb[KS];
    uint32_t q_pb[KS];   // 2^b (0 for a lane without a mission): the tabu-bit shift as a multiplication
#pragma unroll
    for (int k = 0; k < KS; k++) {
        const int m2 = lo + lane + 32 * k;
        int d2 = 0, e2 = W.tdtsm, p2 = tsm, w2 = 0, dep2 = 0, kb = 0, ws2 = NEG, slk = 0, bf = 0xFFFF;
        uint32_t tb = 0;
        q_s2[k] = -1;
        if (m2 >= 0) {
            if (!SV) q_s2[k] = LK[m2] & 0xFFFF;
            const int4 r2 = RS4[m2];
            const int b = (int16_t)((uint32_t)r2.w >> 16);
            if (b >= 0) {
                const int4 c2 = CS4[m2];
                const uint32_t vc = VC[b];
                const int cb = vc & 0xFF;
                const int s2 = LK[m2] & 0xFFFF;
                const int4 rs2 = RS4[s2];
                const int4 cs2 = CS4[s2];
                d2 = 2 * (int)((uint32_t)c2.y >> 16);                       // column del2 of Tt (row pick(s1))
                e2 = W.tdtsm + 2 * (cb * n * NLp + (r2.w & 0xFFFF));         // TDT_cb column endc2 (row m1)
                p2 = tsm + 2 * (cb * NL * NLp + (cs2.y & 0xFFFF));          // column pick(s2) of T_cb (row del1)
                w2 = c2.x;
                dep2 = r2.x;
                kb = rs2.z - r2.y - rs2.y;                                  // svco(s2) - inc2 - inc(s2)
                ws2 = cs2.x - rs2.z;                                        // w(s2) - svco(s2)
                slk = (P - C.F[b]) - (((vc >> 8) & 1) ? 0 : WIN_HELI_OFF);
                bf = b | (MH[m2] ? (int)0x80000000 : 0);
                if (TABU) tb = W.TB[m2];
            }
        }
        q_d2[k] = d2; q_e2[k] = e2; q_p2[k] = p2; q_w2[k] = w2; q_dep2[k] = dep2;
        q_kb[k] = kb; q_ws2[k] = ws2; q_slk[k] = slk; q_bf[k] = bf; q_tb[k] = tb;
        q_pb[k] = (bf & 0xFFFF) < 32 ? 1u << (bf & 0xFFFF) : 0u;
    }
    const int mlane = lo + lane;   // m2 of sub-chunk 0 (sub-chunk k: + 32 k)
    const int NLp2 = 2 * NLp;
    uint64_t best = KEY_NONE;
    for (int w0 = m1_lo; w0 < m1_hi; w0 += WIN_ROWS) {
        __syncwarp();
        if (w0 + lane < m1_hi) win_swap_record<TABU, SV>(C, W, w0 + lane, lane, tsm, asp);
        __syncwarp();
        const int nr = min(WIN_ROWS, m1_hi - w0);
        uint32_t bk = WIN_NONE;
        // One row m1 = w0 + r.  TRIM0 / TRIM1: sub-chunk k may hold m2 <= m1 (the triangle test is
        // needed); SKIP0: sub-chunk 0 lies entirely on or below the diagonal.  Rows below lo need no
        // triangle test at all, so the row loop is split into three ranges with their own bodies.
        // row terms that depend on m1 = w0 + r, formed from r by one add / IMAD each
        const int rowM1_w0 = w0 * NLp2;          // TDT row offset of m1 = w0
        const int trim_w0 = mlane - 1 - w0;      // m2 - m1 - 1 of sub-chunk 0 at m1 = w0
        auto row = [&](int r, auto TRIM0, auto TRIM1, auto SKIP0) {
            const int4 *rec = W.WB + r * WIN_REC_INT4;
            const int4 q2 = rec[2];
            const int hmask = q2.w;
            const int4 q0 = rec[0], q1 = rec[1];
            const int cmask = q0.x, a = q0.x & 0x3F, row_ya1 = q0.y, row_ta2 = q0.z, rowD = q0.w;
            const int s1 = (q0.x >> 8) & 0x7FFF;
            const int ndepc1 = q1.x, w1 = q1.y, wsv1 = q1.z, ka = q1.w;
            const int slkA = q2.x, keyb0 = q2.y;
            const uint32_t tb1 = (uint32_t)q2.z;
            const uint32_t pa = 1u << a;   // a < 32 (window path: V <= 32)
            const int rowM1 = madd(r, NLp2, rowM1_w0);   // TDT row m1 (2 m1 NLp)
            const uint32_t ya_base = (uint32_t)madd(mlane, 2, row_ya1);   // TD_ca[endc1][m2 of sub-chunk 0]
#pragma unroll
            for (int k = 0; k < KS; k++) {
                if (k == 0 && decltype(SKIP0)::value) continue;
                const bool trim_k = k ? decltype(TRIM1)::value : decltype(TRIM0)::value;
                const int bf = q_bf[k];
                const uint32_t b = (uint32_t)bf & 0xFFFFu;
                static_assert(KS == 2, "immediate offsets below assume two sub-chunks");
                const int ya1 = k ? lds_u16_off<64>(ya_base) : lds_u16_off<0>(ya_base);     // d_a(p1, m2)
                const int Ta2 = lds_t<uint16_t>((uint32_t)madd(row_ta2, one, q_d2[k]));     // T_ca[del2][pick(s1)]
                const int yb1 = lds_t<uint16_t>((uint32_t)madd(q_e2[k], one, rowM1));       // d_b(p2, m1)
                const int Tb2 = lds_t<uint16_t>((uint32_t)madd(q_p2[k], one, rowD));        // T_cb[del1][pick(s2)]
                const int da = ya1 + Ta2 + ka;
                const int db = yb1 + Tb2 + q_kb[k];
                const int delta = madd(da, one, db);
                const int mfA = madd(da, neg, slkA);                                        // F_a + da <= P
                const int mfB = madd(db, neg, q_slk[k] & hmask);                            // F_b + db <= P (+ heli)
                const int l1 = madd(ya1, neg, madd(q_w2[k], one, ndepc1));                  // dep(p1) + ya1 <= w2
                const int l2 = wsv1 - q_w2[k] - Ta2;                                        // w2 + d(m2,s1) <= w(s1)
                const int l3 = w1 - q_dep2[k] - yb1;                                        // dep(p2) + yb1 <= w1
                const int l4 = q_ws2[k] - w1 - Tb2;                                         // w1 + d(m1,s2) <= w(s2)
                const int tc = trim_k ? (trim_w0 + 32 * k - r) | (bf & cmask)               // m2 - m1 - 1 >= 0
                                      : (bf & cmask);
                int mg;
                if (SV) {
                    mg = (l1 | l2 | l3) | (l4 | mfA | mfB) | tc;
                } else {   // general legs: same-route flight limit, explicit adjacent pairs
                    const int m1 = w0 + r, m2 = mlane + 32 * k;
                    const int mf = (int)b == a ? madd(delta, neg, slkA) : (mfA | mfB);   // F_a + delta <= P
                    const int adj = (s1 == m2) | (q_s2[k] == m1) ? -1 : 0;
                    mg = (l1 | l2 | l3) | (l4 | mf | adj) | tc;
                }
                uint32_t k32;                                                               // delta holds delta - asp
                if (F1 && SV) {   // see score_reloc_win
                    const uint32_t nz = TABU ? (mul_fma(tb1, q_pb[k]) | mul_fma(q_tb[k], pa)) & ~(uint32_t)delta
                                             : ~(uint32_t)delta;
                    k32 = (uint32_t)madd(delta, 1 << WIN_KEY_SHIFT, keyb0 + k) | ((nz | (uint32_t)mg) & 0x80000000u);
                } else {
                    uint32_t nadm;
                    if (TABU) nadm = (mul_fma(tb1, q_pb[k]) | mul_fma(q_tb[k], pa)) & ~(uint32_t)delta & 0x80000000u;
                    else nadm = ~(uint32_t)delta & 0x80000000u;
                    k32 = (uint32_t)madd(delta, 1 << WIN_KEY_SHIFT, keyb0 + k) | nadm | (uint32_t)(mg >> 31);
                }
                bk = min(bk, k32);
            }
        };
        using F_ = std::integral_constant<bool, false>;
        using T_ = std::integral_constant<bool, true>;
        const int e1 = max(0, min(nr, lo - w0)), e2 = max(e1, min(nr, lo + 31 - w0));
        for (int r = 0; r < e1; r++) row(r, F_{}, F_{}, F_{});    // m1 < lo: every lane above the diagonal
        for (int r = e1; r < e2; r++) row(r, T_{}, F_{}, F_{});   // diagonal band of sub-chunk 0
        for (int r = e2; r < nr; r++) row(r, F_{}, T_{}, T_{});   // sub-chunk 0 done; band of sub-chunk 1
        if (bk != WIN_NONE) {
            const int lid = bk & ((1 << WIN_KEY_SHIFT) - 1);
            const uint32_t idx = Rb + (uint32_t)(w0 + lid / KS) * (uint32_t)n + (uint32_t)(lo + lane + 32 * (lid % KS));
            const uint64_t key = win_key64(bk, idx);
            best = key < best ? key : best;
        }
    }
    return best;
}

}  // namespace airsched
