// score.cuh -- the per-move scoring loops of the evaluation kernels (sm_100a).
//
// A "tile" is a set of moves one warp scores with part of the operands cached
// in registers: a relocate tile is one chunk of 32*KR target slots (the
// target-side records are cached per lane) times a range of rows m; a swap tile
// is one chunk of 32*KS missions m2 aligned to the top of [0, n) (the m2-side
// records are cached per lane) times a range of rows m1 < m2.  Inside a tile a
// lane visits its moves in increasing canonical index, so the per-lane best is
// kept as a 32-bit key (class << 31 | delta + 2^30) plus the index, and a strict
// '<' keeps the lowest index among equal keys (O9, reading #26).  Each scorer
// returns the tile's best packed 64-bit key for this lane (AS_KEY_NONE if none).
//
// Table reads: every scored move reads T at (row x, column y) with one of x, y
// fixed for the whole row m (m1) and the other varying over the lanes.  With the
// table in shared memory (TR = false) the lanes read down a column (rows spread
// over the banks by the odd padded stride).  With the table in global memory
// (TR = true) the lanes read along ONE row -- of T, or of its per-layer
// transpose Tt -- so each row m touches a few L1-resident rows shared by the
// CTA's warps instead of a different row per lane.
//
// Formulas: DESIGN.md §3 (the same arithmetic as engine.cuh, rewritten for
// register-resident operands; adjacent swaps are excluded here and scored by
// engine.cuh's exact three-link formula).  Operands are in the AoS records of
// batch.cu's layout (CS: per-slot constants, RS: per-slot incoming-link record,
// LK: links), in shared or global memory.
#pragma once
#include <cstdint>

#include "engine.cuh"

namespace airsched {

constexpr int KR = 4;              // relocate tile: 4 x 32 target slots cached per lane
constexpr int KS = 2;              // swap tile: 2 x 32 m2 missions cached per lane
constexpr int NEG = -(1 << 29);    // "never feasible" margin

// Integer adds and selects on the FMA pipe.  Blackwell issues IADD3 / LOP3 /
// ISETP / SEL / VIMNMX on the ALU pipe and IMAD on the FMA pipe, each at half
// rate (B300_MICROARCH.md, "fma vs alu split"); the scoring loops saturate the
// ALU pipe (profiles/r01), so sums are written as mad.lo.s32 with a multiplier
// the compiler cannot prove to be 1 (ScoreCtx::one == 1, ScoreCtx::neg == -1 at
// run time) and land on the otherwise idle FMA pipe.  Exact integer results.
__device__ __forceinline__ int madd(int a, int mul, int b) {   // a * mul + b
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(mul), "r"(b));
    return r;
}

// Shared-memory table read at a 32-bit shared-window byte address (the FAST
// scorers fold the table base and the element size into their cached offsets,
// so one integer add forms each address).
template <class TT>
__device__ __forceinline__ int lds_t(uint32_t addr);
template <>
__device__ __forceinline__ int lds_t<uint16_t>(uint32_t addr) {
    unsigned short v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return (int)v;
}
template <>
__device__ __forceinline__ int lds_t<int32_t>(uint32_t addr) {
    int v;
    asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

template <class TT, class ET>
struct ScoreCtx {
    const TT *Ts;          // [NC][NL][NLp] travel times
    const TT *Tt;          // the same, transposed per layer (== Ts for symmetric tables)
    const int4 *CS4;       // [S] {w, pick | del << 16, svc0, svc1}
    const uint8_t *MH;     // [n] helicopter-only
    const uint32_t *VC;    // [V] cls | heli_ok << 8 | base location << 16
    const int4 *RS4;       // [S] {depc, inc, svco, endc | veh << 16}
    const uint32_t *LK;    // [S] succ | pred << 16
    const int32_t *F;      // [V] route flight time
    const ET *E;           // [n][V] tabu expiry (TABU only)
    const ET *Et;          // [V][n] its transpose when E is in global memory (row-local E[m2][a] reads), else null
    const uint16_t *TD;    // global-table scorers (TR): node costs TD[c][x][t] (DevInst::TDg), else null
    const int2 *RR;        // FAST relocate rows cached per CTA (k_grid, global table): {a, or -1 when the row has
                           // no feasible relocate; removal delta rem} -- see reloc_row_record; or null
    int4 *SR;              // FAST swap rows, per-warp scratch (k_grid, global table): SR_ROWS x 2 int4 per warp,
                           // filled lane-parallel at the start of each tile -- see score_swap_fast; or null
    int n, V, S, NL, NLp, P;
    uint32_t Rb, mask;
    int one, neg;          // 1 and -1, opaque to the compiler (see madd)
};

template <bool TABU, bool FULL, bool TR = false, class TT, class ET>
__device__ __forceinline__ uint64_t score_reloc(const ScoreCtx<TT, ET> &C, int t0, int m_lo, int m_hi, int it,
                                                int asp, int lane) {
    const TT *Ts = C.Ts, *Tt = C.Tt;
    const int4 *CS4 = C.CS4, *RS4 = C.RS4;
    const uint8_t *MH = C.MH;
    const uint32_t *VC = C.VC, *LK = C.LK;
    const int32_t *F = C.F;
    const ET *E = C.E;
    const int V = C.V, S = C.S, NL = C.NL, NLp = C.NLp, P = C.P;
    const uint32_t mask = C.mask;
    const bool en_inter_r = FULL || (mask & 1u) != 0, en_intra_r = FULL || (mask & 2u) != 0;
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
                t1 = TR ? cb * NL * NLp + (rs.w & 0xFFFF)    // column endc(t) of Tt_cb (row pick_m per m)
                        : (cb * NL + (rs.w & 0xFFFF)) * NLp; // row endc(t) of T_cb (column pick_m per m)
                t2 = cb * NL * NLp + (cs.y & 0xFFFF);        // column pick(t) of T_cb (row del_m per m)
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
    for (int m = m_lo; m < m_hi; m++) {
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
        const int w_m = cm.x, rowP = TR ? (cm.y & 0xFFFF) * NLp : (cm.y & 0xFFFF), rowD = ((uint32_t)cm.y >> 16) * NLp;
        const int svm0 = cm.z, svm1 = cm.w;
        const bool heli_m = MH[m] != 0;
        const ET *Erow = TABU ? E + m * V : nullptr;
        const uint32_t base = (uint32_t)m * (uint32_t)S + t0 + lane;
        const int one = C.one, neg = C.neg;
        const int wm_neg = madd(w_m, neg, 0);                      // -w_m
#pragma unroll
        for (int k = 0; k < KR; k++) {
            const int t = t0 + lane + 32 * k;
            const int inf = c_inf[k];
            const int b = (int)(int16_t)(inf & 0xFFFF);
            const bool cb1 = (inf >> 16) & 1;
            const bool hok = (inf >> 20) & 1;
            const int T1 = (int)(TR ? Tt : Ts)[madd(c_t1[k], one, rowP)];     // T_cb[endc t][pick m]
            const int T2 = (int)Ts[madd(c_t2[k], one, rowD)];     // T_cb[del m][pick t]
            const int x1 = madd(T1, one, cb1 ? svm1 : svm0);
            const int ins = madd(x1, one, madd(T2, one, c_k[k]));
            const int delta = madd(rem, one, ins);
            const bool same = b == a;
            const int lim = same ? intra_lim : madd(c_slk[k], one, inter_bias);
            const int mg = min(min(madd(x1, neg, madd(w_m, one, c_dw[k])), madd(T2, neg, madd(c_wsv[k], one, wm_neg))),
                               madd(ins, neg, lim));
            const bool ok = (mg >= 0) & (t != m) & (t != s) & (FULL || (same ? en_intra_r : en_inter_r)) &
                            (hok | !heli_m);
            bool adm;
            if (TABU) adm = ((int)Erow[max(b, 0)] < it) | (delta < asp);
            else adm = delta < 0;
            uint32_t k32 = (uint32_t)madd(delta, one, DELTA_BIAS) | (adm ? 0u : 0x80000000u);
            k32 = ok ? k32 : 0xFFFFFFFFu;
            const bool better = k32 < bk32;
            bk32 = better ? k32 : bk32;
            bidx = better ? base + 32 * k : bidx;
        }
    }    return bk32 == 0xFFFFFFFFu ? KEY_NONE : (((uint64_t)bk32 << 32) | bidx);
}

template <bool TABU, bool FULL, bool TR = false, class TT, class ET>
__device__ __forceinline__ uint64_t score_swap(const ScoreCtx<TT, ET> &C, int hi, int m1_lo, int m1_hi, int it,
                                               int asp, int lane) {
    const TT *Ts = C.Ts, *Tt = C.Tt;
    const int4 *CS4 = C.CS4, *RS4 = C.RS4;
    const uint8_t *MH = C.MH;
    const uint32_t *VC = C.VC, *LK = C.LK;
    const int32_t *F = C.F;
    const ET *E = C.E;
    const int n = C.n, V = C.V, NL = C.NL, NLp = C.NLp, P = C.P;
    const uint32_t Rb = C.Rb, mask = C.mask;
    const bool en_inter_s = FULL || (mask & 4u) != 0, en_intra_s = FULL || (mask & 8u) != 0;
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
                d2 = TR ? (int)((uint32_t)c2.y >> 16)              // column del2 of Tt (row pick(s1) per m1)
                        : (int)((uint32_t)c2.y >> 16) * NLp;       // row del2 of T (column pick(s1) per m1)
                e2 = TR ? cb * NL * NLp + (r2.w & 0xFFFF)          // column endc2 of Tt_cb (row pick1 per m1)
                        : (cb * NL + (r2.w & 0xFFFF)) * NLp;       // row endc2 of T_cb (column pick1 per m1)
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
    for (int m1 = m1_lo; m1 < m1_hi; m1++) {
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
        const int row_ta2 = TR ? (ca * NL + (cs1.y & 0xFFFF)) * NLp   // Tt_ca[pick(s1)][.]
                               : ca * NL * NLp + (cs1.y & 0xFFFF);    // T_ca[.][pick(s1)]
        const int rowp1 = TR ? (c1.y & 0xFFFF) * NLp : (c1.y & 0xFFFF), row_tb2 = ((uint32_t)c1.y >> 16) * NLp;
        const int depc1 = r1.x, w1 = c1.x;
        const bool heli1 = MH[m1] != 0;
        const int wsv1 = cs1.x - rs1.z;                 // w(s1) - svco(s1)
        const int ka = rs1.z - r1.y - rs1.y;            // svco(s1) - inc1 - inc(s1)
        const int slkA = P - F[a];
        const int sv10 = c1.z, sv11 = c1.w;
        const ET *Erow = TABU ? E + m1 * V : nullptr;
        // E[m2][a] over the lanes: a column of E, or (global tables, TR) a row of its transpose
        const ET *ecol = TABU ? ((TR && C.Et) ? C.Et + (size_t)a * C.n : E + a) : nullptr;
        const int estr = (TR && C.Et) ? 1 : V;
        const uint32_t base = Rb + (uint32_t)m1 * (uint32_t)n + lo + lane;
        const int one = C.one, neg = C.neg;
        const int ndepc1 = madd(depc1, neg, 0), nw1 = madd(w1, neg, 0);
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
            const int ya1 = madd((int)Ts[madd(row_ya1, one, pick2)], one, ca ? q_sv1[k] : q_sv0[k]); // p1 -> m2
            const int Ta2 = (int)(TR ? Tt : Ts)[madd(row_ta2, one, q_d2[k])];                              // m2 -> s1
            const int yb1 = madd((int)(TR ? Tt : Ts)[madd(q_e2[k], one, rowp1)], one, cb1 ? sv11 : sv10);  // p2 -> m1
            const int Tb2 = (int)Ts[madd(q_p2[k], one, row_tb2)];                             // m1 -> s2
            const int da = madd(ya1, one, madd(Ta2, one, ka));
            const int db = madd(yb1, one, madd(Tb2, one, q_kb[k]));
            const int delta = madd(da, one, db);
            const int mA = madd(da, neg, slkA), mB = madd(db, neg, q_slk[k]);
            const int mf = same ? madd(delta, neg, slkA) : min(mA, mB);
            const int mg = min(min(min(madd(ya1, neg, madd(q_w2[k], one, ndepc1)),
                                       madd(Ta2, neg, madd(q_w2[k], neg, wsv1))),
                                   min(madd(yb1, neg, madd(q_dep2[k], neg, w1)),
                                       madd(Tb2, neg, madd(q_ws2[k], one, nw1)))),
                               mf);
            const bool ok = (mg >= 0) & (m2 > m1) & (s1 != m2) & (s2 != m1) &
                            (FULL || (same ? en_intra_s : en_inter_s)) & (!h2 | hoka) & (!heli1 | hokb);
            bool adm;
            if (TABU) adm = (((int)Erow[max(b, 0)] < it) & ((int)ecol[max(m2, 0) * estr] < it)) | (delta < asp);
            else adm = delta < 0;
            uint32_t k32 = (uint32_t)madd(delta, one, DELTA_BIAS) | (adm ? 0u : 0x80000000u);
            k32 = ok ? k32 : 0xFFFFFFFFu;
            const bool better = k32 < bk32;
            bk32 = better ? k32 : bk32;
            bidx = better ? base + 32 * k : bidx;
        }
    }    return bk32 == 0xFFFFFFFFu ? KEY_NONE : (((uint64_t)bk32 << 32) | bidx);
}

// ---------------------------------------------------------------------------
// FAST scorers: every move kind enabled AND every pickup->delivery leg > 0 in
// every class (DevInst::svcpos).  Then the two no-op relocate targets (t = m,
// t = succ m) and the adjacent swap pairs fail a link check by construction
// (their margins are -svc < 0), so no per-move validity test is
// needed; and every intra-route move fails one of its new-link checks (a
// feasible route is strictly deadline-sorted, reading #42), so the flight
// limit is checked in its inter-route form for every move and a relocate row
// whose removal leaves route a over the limit is skipped.  Feasibility,
// compatibility and the triangle m1 < m2 are OR-combined into one margin whose
// sign bit poisons the key, admissibility is a sign-bit expression, and sums are
// split between 3-input adds (ALU pipe) and mad.lo (FMA pipe) -- the scoring
// loops are issue-bound, so every instruction removed counts.
//
// Global tables (TR) are read through the read-only data path (__ldg: the table never changes
// during a run).
// Keys: with a uint16 table (|delta| < 2^20) a lane keeps the 32-bit key
// nadm << 31 | (delta + 2^23) << 7 | local index over blocks of 32 rows (one
// unsigned min per move, the index recovered at the block's end, window.cuh);
// with an int32 table it keeps (class << 31 | delta + 2^30) and the index.
constexpr int FB_ROWS = 32;   // rows per key block (uint16 tables)
constexpr int SR_ROWS = 16;   // swap rows per per-warp record batch (ScoreCtx::SR)

template <bool TABU, bool TR = false, class TT, class ET>
__device__ __forceinline__ uint64_t score_reloc_fast(const ScoreCtx<TT, ET> &C, int t0, int m_lo, int m_hi, int it,
                                                     int asp, int lane) {
    constexpr bool K16 = sizeof(TT) == 2;
    const TT *Ts = C.Ts, *Tt = C.Tt;
    const int4 *CS4 = C.CS4, *RS4 = C.RS4;
    const uint8_t *MH = C.MH;
    const uint32_t *VC = C.VC, *LK = C.LK;
    const int32_t *F = C.F;
    const ET *E = C.E;
    const int V = C.V, S = C.S, NL = C.NL, NLp = C.NLp, P = C.P;
    // global tables (TR): every table read adds an IMAD.WIDE on the FMA pipe, which then saturates first --
    // the sums go back to the ALU pipe there (one and neg known to the compiler)
    const int one = TR ? 1 : C.one, neg = TR ? -1 : C.neg;
    int c_t1[KR], c_t2[KR], c_dw[KR], c_k[KR], c_wsv[KR], c_slk[KR], c_b[KR], c_cb[KR];
    // shared table (TR false): cached offsets are byte addresses in the shared window
    const int tsm = TR ? 0 : (int)__cvta_generic_to_shared(Ts), tsz = TR ? 1 : (int)sizeof(TT);
    // global table with node costs (TR, uint16): d_b(m, t) = T_cb[del_m][pick_t] + svco(t) is ONE read of
    // TD_cb row del_m at column t -- consecutive lanes, consecutive slots: a coalesced 64-byte read
    // instead of a gather over the row
    const bool td = TR && K16 && C.TD != nullptr;
    const TT *T2p = td ? reinterpret_cast<const TT *>(C.TD) : Ts;
    const int tdS = td ? S : NLp;
#pragma unroll
    for (int k = 0; k < KR; k++) {
        const int t = t0 + lane + 32 * k;
        int t1 = tsm, t2 = tsm, dw = 0, kk = 0, wsv = NEG, slk = 0, b = 0, cb = 0;
        if (t < S) {
            const int4 rs = RS4[t];
            const int bb = (int16_t)((uint32_t)rs.w >> 16);
            if (bb >= 0) {
                const int4 cs = CS4[t];
                const uint32_t vc = VC[bb];
                b = bb;
                cb = vc & 0xFF;
                t1 = TR ? cb * NL * NLp + (rs.w & 0xFFFF)    // column endc(t) of Tt_cb (row pick_m per m)
                        : tsm + tsz * ((cb * NL + (rs.w & 0xFFFF)) * NLp); // row endc(t) of T_cb (column pick_m)
                t2 = td ? cb * NL * S + t                          // column t of TD_cb (row del_m per m)
                        : tsm + tsz * (cb * NL * NLp + (cs.y & 0xFFFF)); // column pick(t) of T_cb (row del_m per m)
                dw = -rs.x;                                  // -dep(pred t)
                kk = td ? -rs.y : rs.z - rs.y;               // svco(t) - inc(t) (TD: svco(t) is in the node cost)
                wsv = td ? cs.x : cs.x - rs.z;               // w(t) - svco(t)
                slk = (P - F[bb]) - (((vc >> 8) & 1) ? 0 : (1 << 30));   // heli offset (masked off for non-heli rows)
            }
        }
        c_t1[k] = t1; c_t2[k] = t2; c_dw[k] = dw; c_k[k] = kk; c_wsv[k] = wsv; c_slk[k] = slk; c_b[k] = b;
        c_cb[k] = cb;
    }
    uint64_t best = KEY_NONE;
    uint32_t bk32 = 0xFFFFFFFFu, bidx = 0;
    for (int m0 = m_lo; m0 < m_hi; m0 += FB_ROWS) {
        const int m_end = min(m_hi, m0 + FB_ROWS);
        if (K16) bk32 = 0xFFFFFFFFu;
        for (int m = m0; m < m_end; m++) {
            int rem;
            if (TR && C.RR) {   // the row's removal side, cached per CTA and refreshed after every move
                const int2 rr = C.RR[m];
                if (rr.x < 0) continue;
                rem = rr.y;
            } else {
                const int4 rm = RS4[m];
                const int a = (int16_t)((uint32_t)rm.w >> 16);
                if (a < 0) continue;
                const int s = LK[m] & 0xFFFF;
                const int4 rsx = RS4[s];
                const int4 csx = CS4[s];
                const int ca = VC[a] & 0xFF;
                const int Dps = (int)Ts[(ca * NL + (rm.w & 0xFFFF)) * NLp + (csx.y & 0xFFFF)] + rsx.z;
                if (rm.x + Dps > csx.x) continue;     // link p->s infeasible: every relocate of m is
                rem = Dps - rm.y - rsx.y;
                if (F[a] + rem > P) continue;         // no feasible relocate of m (reading #42)
            }
            const int4 cm = CS4[m];
            const int w_m = cm.x, rowP = TR ? (cm.y & 0xFFFF) * NLp : tsz * (cm.y & 0xFFFF),
                      rowD = tsz * (int)((uint32_t)cm.y >> 16) * tdS;
            const int svm0 = cm.z, dsvm = cm.w - cm.z, wm_neg = -cm.x;
            const int hmask = MH[m] ? (int)0xFFFFFFFF : 0x3FFFFFFF;
            const int remasp = TABU ? rem - asp : rem;
            const uint32_t erow = (uint32_t)(m * V);   // 32-bit element index: one IMAD.WIDE per tabu read
            const int remk = (rem + (1 << 23)) * 128 + (m - m0) * KR;            // K16 key base
            const uint32_t base = (uint32_t)m * (uint32_t)S + t0 + lane;        // int32-table index
#pragma unroll
            for (int k = 0; k < KR; k++) {
                // T_cb[endc t][pick m], T_cb[del m][pick t]; shared table: byte addresses
                const int T1 = TR ? (int)__ldg(&Tt[madd(c_t1[k], one, rowP)]) : lds_t<TT>((uint32_t)madd(c_t1[k], one, rowP));
                const int T2 = TR ? (int)__ldg(&T2p[madd(c_t2[k], one, rowD)]) : lds_t<TT>((uint32_t)madd(c_t2[k], one, rowD));
                const int x1 = madd(c_cb[k], dsvm, madd(T1, one, svm0));              // d(c, m)
                const int ins = x1 + T2 + c_k[k];
                const int mA = madd(x1, neg, madd(w_m, one, c_dw[k]));               // dep(c) + d(c,m) <= w_m
                const int mB = c_wsv[k] + wm_neg - T2;                                // w_m + d(m,t) <= w(t)
                const int mC = madd(ins, neg, c_slk[k] & hmask);                      // F_b + ins <= P (+ heli)
                const int mg = mA | mB | mC;
                const int e2 = madd(ins, one, remasp);                                // delta - asp (TS) / delta (NS)
                uint32_t nadm;
                if (TABU) {
                    const int e1 = madd(it, neg, (int)E[erow + (uint32_t)c_b[k]]);    // E[m][b] - it (>= 0: tabu)
                    nadm = ~(uint32_t)(e1 | e2) & 0x80000000u;
                } else {
                    nadm = ~(uint32_t)e2 & 0x80000000u;
                }
                if constexpr (K16) {
                    const uint32_t k32 = (uint32_t)madd(ins, 128, remk + k) | nadm | (uint32_t)(mg >> 31);
                    bk32 = min(bk32, k32);
                } else {
                    const uint32_t k32 = (uint32_t)madd(rem + ins, one, DELTA_BIAS) | nadm | (uint32_t)(mg >> 31);
                    const bool better = k32 < bk32;
                    bk32 = better ? k32 : bk32;
                    bidx = better ? base + 32 * k : bidx;
                }
            }
        }
        if (K16 && bk32 != 0xFFFFFFFFu) {
            const int lid = bk32 & 127;
            const uint32_t idx = (uint32_t)(m0 + lid / KR) * (uint32_t)S + (uint32_t)(t0 + lane + 32 * (lid % KR));
            const uint32_t d = ((bk32 >> 7) & 0xFFFFFFu) + (uint32_t)(DELTA_BIAS - (1 << 23));
            const uint64_t key = ((uint64_t)((bk32 & 0x80000000u) | d) << 32) | idx;
            best = key < best ? key : best;
        }
    }
    if (!K16) best = bk32 == 0xFFFFFFFFu ? KEY_NONE : (((uint64_t)bk32 << 32) | bidx);
    return best;
}

template <bool TABU, bool TR = false, class TT, class ET>
__device__ __forceinline__ uint64_t score_swap_fast(const ScoreCtx<TT, ET> &C, int hi, int m1_lo, int m1_hi, int it,
                                                    int asp, int lane) {
    constexpr bool K16 = sizeof(TT) == 2;
    const TT *Ts = C.Ts, *Tt = C.Tt;
    const int4 *CS4 = C.CS4, *RS4 = C.RS4;
    const uint8_t *MH = C.MH;
    const uint32_t *VC = C.VC, *LK = C.LK;
    const int32_t *F = C.F;
    const ET *E = C.E;
    const int n = C.n, V = C.V, NL = C.NL, NLp = C.NLp, P = C.P;
    const uint32_t Rb = C.Rb;
    // global tables (TR): every table read adds an IMAD.WIDE on the FMA pipe, which then saturates first --
    // the sums go back to the ALU pipe there (one and neg known to the compiler)
    const int one = TR ? 1 : C.one, neg = TR ? -1 : C.neg;
    const int lo = hi - 32 * KS;
    const int sa = TABU ? asp : 0;   // aspiration folded into route a's terms: "dl" below is delta - asp
    // m2-side cache; q_bf = b | heli_only(m2) << 31; q_slk carries the heli offset
    int q_p2m[KS], q_sv0[KS], q_dsv[KS], q_d2[KS], q_e2[KS], q_p2[KS], q_w2[KS], q_dep2[KS], q_kb[KS], q_ws2[KS],
        q_slk[KS], q_bf[KS];
    int q_cb[KS];
    // shared table (TR false): offsets are byte addresses in the shared window, the base on one side of each pair
    const int tsm = TR ? 0 : (int)__cvta_generic_to_shared(Ts), tsz = TR ? 1 : (int)sizeof(TT);
    // global table with node costs (TR, uint16): d_a(p1, m2) = T_ca[endc1][pick2] + svc_ca(m2) is ONE read of
    // TD_ca row endc1 at column m2 -- consecutive lanes: coalesced
    const bool td = TR && K16 && C.TD != nullptr;
    const TT *Tyap = td ? reinterpret_cast<const TT *>(C.TD) : Ts;
    const int S = n + V, tdS = td ? S : NLp;
#pragma unroll
    for (int k = 0; k < KS; k++) {
        const int m2 = lo + lane + 32 * k;
        int p2m = 0, sv0 = 0, dsv = 0, d2 = 0, e2 = tsm, p2 = tsm, w2 = 0, dep2 = 0, kb = 0, ws2 = NEG, slk = 0,
            bf = 0, cb = 0;
        if (m2 >= 0) {
            const int4 r2 = RS4[m2];
            const int b = (int16_t)((uint32_t)r2.w >> 16);
            if (b >= 0) {
                const int4 c2 = CS4[m2];
                const uint32_t vc = VC[b];
                cb = vc & 0xFF;
                const int s2 = LK[m2] & 0xFFFF;
                const int4 rs2 = RS4[s2];
                const int4 cs2 = CS4[s2];
                p2m = td ? m2 : tsz * (c2.y & 0xFFFF);            // pick2 (TD: column m2)
                sv0 = td ? 0 : c2.z;
                dsv = td ? 0 : c2.w - c2.z;
                d2 = TR ? (int)((uint32_t)c2.y >> 16)              // column del2 of Tt (row pick(s1) per m1)
                        : tsz * (int)((uint32_t)c2.y >> 16) * NLp; // row del2 of T (column pick(s1) per m1)
                e2 = TR ? cb * NL * NLp + (r2.w & 0xFFFF)          // column endc2 of Tt_cb (row pick1 per m1)
                        : tsm + tsz * ((cb * NL + (r2.w & 0xFFFF)) * NLp); // row endc2 of T_cb (column pick1)
                p2 = tsm + tsz * (cb * NL * NLp + (cs2.y & 0xFFFF)); // column pick(s2) of T_cb
                w2 = c2.x;
                dep2 = r2.x;
                kb = rs2.z - r2.y - rs2.y;                        // svco(s2) - inc2 - inc(s2)
                ws2 = cs2.x - rs2.z;                              // w(s2) - svco(s2)
                slk = (P - F[b]) - (((vc >> 8) & 1) ? 0 : (1 << 30));
                bf = b | (MH[m2] ? (int)0x80000000 : 0);
            }
        }
        q_p2m[k] = p2m; q_sv0[k] = sv0; q_dsv[k] = dsv; q_d2[k] = d2; q_e2[k] = e2; q_p2[k] = p2; q_w2[k] = w2;
        q_dep2[k] = dep2; q_kb[k] = kb; q_ws2[k] = ws2; q_slk[k] = slk; q_bf[k] = bf; q_cb[k] = cb;
    }
    const int mlane = lo + lane;
    uint64_t best = KEY_NONE;
    uint32_t bk32 = 0xFFFFFFFFu, bidx = 0;
    // E[m2][a] over the lanes: a column of E, or (global tables, TR) a row of its transpose
    const ET *ecol = TABU ? ((TR && C.Et) ? C.Et : E) : nullptr;
    const uint32_t estr = (TR && C.Et) ? 1u : (uint32_t)V;
    // the row side of m1 (route a, successor s1): its dynamic part either computed here by the whole warp, or
    // (TR && C.SR) computed once per row by one lane into the warp's record scratch at the start of each batch
    int4 *SRw = (TR && C.SR) ? C.SR + (threadIdx.x >> 5) * (2 * SR_ROWS) : nullptr;
    auto row_side = [&](int m1, int &a, int &ca, int &row_ya1, int &row_ta2, int &ndepc1, int &wsv1, int &ka,
                        int &slkA, int &cmask, int &hmask) {
        const int4 r1 = RS4[m1];
        a = (int16_t)((uint32_t)r1.w >> 16);
        if (a < 0) return;
        const int s1 = LK[m1] & 0xFFFF;
        const int4 rs1 = RS4[s1];
        const int4 cs1 = CS4[s1];
        const uint32_t vca = VC[a];
        ca = vca & 0xFF;
        row_ya1 = tsm + tsz * ((ca * NL + (r1.w & 0xFFFF)) * tdS);      // T_ca[endc1][.] (TD_ca[endc1][.])
        row_ta2 = TR ? (ca * NL + (cs1.y & 0xFFFF)) * NLp                // Tt_ca[pick(s1)][.]
                     : tsm + tsz * (ca * NL * NLp + (cs1.y & 0xFFFF));   // T_ca[.][pick(s1)]
        ndepc1 = -r1.x;
        wsv1 = cs1.x - rs1.z;                 // w(s1) - svco(s1)
        ka = rs1.z - r1.y - rs1.y - sa;       // svco(s1) - inc1 - inc(s1) - asp
        slkA = P - F[a] - sa;
        cmask = ((vca >> 8) & 1) ? 0 : (int)0x80000000;   // route a cannot fly heli-only missions
        hmask = MH[m1] ? (int)0xFFFFFFFF : 0x3FFFFFFF;
    };
    for (int w0 = m1_lo; w0 < m1_hi; w0 += FB_ROWS) {
        const int w_end = min(m1_hi, w0 + FB_ROWS);
        if (K16) bk32 = 0xFFFFFFFFu;
        for (int m1 = w0; m1 < w_end; m1++) {
            int a = -1, ca = 0, row_ya1 = 0, row_ta2 = 0, ndepc1 = 0, wsv1 = 0, ka = 0, slkA = 0, cmask = 0, hmask = 0;
            if (TR && SRw) {
                const int j = (m1 - w0) % SR_ROWS;
                if (j == 0) {   // next batch of rows: one lane per row
                    __syncwarp();
                    const int mr = m1 + lane;
                    if (lane < SR_ROWS && mr < w_end) {
                        row_side(mr, a, ca, row_ya1, row_ta2, ndepc1, wsv1, ka, slkA, cmask, hmask);
                        SRw[2 * lane] = make_int4(row_ya1, row_ta2, ndepc1, wsv1);
                        SRw[2 * lane + 1] = make_int4(ka, slkA, a, ca | (cmask ? 0x100 : 0) | (hmask == -1 ? 0x200 : 0));
                    }
                    __syncwarp();
                }
                const int4 x0 = SRw[2 * j], x1 = SRw[2 * j + 1];
                a = x1.z;
                if (a < 0) continue;
                row_ya1 = x0.x; row_ta2 = x0.y; ndepc1 = x0.z; wsv1 = x0.w;
                ka = x1.x; slkA = x1.y;
                ca = x1.w & 0xFF;
                cmask = (x1.w & 0x100) ? (int)0x80000000 : 0;
                hmask = (x1.w & 0x200) ? (int)0xFFFFFFFF : 0x3FFFFFFF;
            } else {
                row_side(m1, a, ca, row_ya1, row_ta2, ndepc1, wsv1, ka, slkA, cmask, hmask);
                if (a < 0) continue;
            }
            const int4 c1 = CS4[m1];
            const int rowp1 = TR ? (c1.y & 0xFFFF) * NLp : tsz * (c1.y & 0xFFFF);
            const int row_tb2 = tsz * (int)((uint32_t)c1.y >> 16) * NLp;
            const int w1 = c1.x;
            const int sv10 = c1.z, dsv1 = c1.w - c1.z;
            const uint32_t erow = (uint32_t)(m1 * V);   // 32-bit element indices: one IMAD.WIDE per tabu read
            const uint32_t ecol0 = (TR && C.Et) ? (uint32_t)a * (uint32_t)C.n : (uint32_t)a;
            const int keyb = (1 << 30) + sa * 128 + (m1 - w0) * KS;               // K16: (2^23 + asp) << 7 | lid
            const uint32_t base = Rb + (uint32_t)m1 * (uint32_t)n + lo + lane;   // int32 tables
#pragma unroll
            for (int k = 0; k < KS; k++) {
                // sub-chunk entirely on or below the diagonal: skipped on the shared-table path; the global-table
                // path scores it masked (trim < 0), so that the loads of both sub-chunks issue back to back
                if (!TR && lo + 32 * k + 31 <= m1) continue;
                const int bf = q_bf[k];
                const int b = bf & 0xFFFF;
                const int a_ya1 = madd(row_ya1, one, q_p2m[k]), a_ta2 = madd(row_ta2, one, q_d2[k]);
                const int a_yb1 = madd(q_e2[k], one, rowp1), a_tb2 = madd(q_p2[k], one, row_tb2);
                const int Tya1 = TR ? (int)__ldg(&Tyap[a_ya1]) : lds_t<TT>((uint32_t)a_ya1);
                const int Ta2 = TR ? (int)__ldg(&Tt[a_ta2]) : lds_t<TT>((uint32_t)a_ta2);                  // m2 -> s1
                const int Tyb1 = TR ? (int)__ldg(&Tt[a_yb1]) : lds_t<TT>((uint32_t)a_yb1);
                const int Tb2 = TR ? (int)__ldg(&Ts[a_tb2]) : lds_t<TT>((uint32_t)a_tb2);                  // m1 -> s2
                const int ya1 = madd(q_dsv[k], ca, madd(Tya1, one, q_sv0[k]));                    // p1 -> m2
                const int yb1 = madd(q_cb[k], dsv1, madd(Tyb1, one, sv10));                       // p2 -> m1
                const int da = ya1 + Ta2 + ka;                                                    // (- asp)
                const int db = yb1 + Tb2 + q_kb[k];
                const int dl = madd(da, one, db);                                                 // delta - asp
                const int mfA = madd(da, neg, slkA);                                              // F_a + da <= P
                const int mfB = madd(db, neg, q_slk[k] & hmask);                                  // F_b + db <= P
                const int l1 = madd(ya1, neg, madd(q_w2[k], one, ndepc1));                        // dep(p1) + ya1 <= w2
                const int l2 = wsv1 - q_w2[k] - Ta2;                                              // w2 + d(m2,s1) <= w(s1)
                const int l3 = w1 - q_dep2[k] - yb1;                                              // dep(p2) + yb1 <= w1
                const int l4 = q_ws2[k] - w1 - Tb2;                                               // w1 + d(m1,s2) <= w(s2)
                const int trim = mlane + (32 * k - 1) - m1;                                       // m2 - m1 - 1 >= 0
                const int mg = (l1 | l2 | l3) | (l4 | mfA | mfB) | (trim | (bf & cmask));
                uint32_t nadm;
                if (TABU) {
                    const int t1 = madd(it, neg, (int)E[erow + (uint32_t)b]);                    // E[m1][b] - it
                    const int t2 = madd(it, neg, (int)ecol[ecol0 + (uint32_t)max(mlane + 32 * k, 0) * estr]);  // E[m2][a] - it
                    nadm = ~(uint32_t)((t1 & t2) | dl) & 0x80000000u;
                } else {
                    nadm = ~(uint32_t)dl & 0x80000000u;
                }
                if constexpr (K16) {
                    const uint32_t k32 = (uint32_t)madd(dl, 128, keyb + k) | nadm | (uint32_t)(mg >> 31);
                    bk32 = min(bk32, k32);
                } else {
                    const uint32_t k32 = (uint32_t)madd(dl, one, DELTA_BIAS + sa) | nadm | (uint32_t)(mg >> 31);
                    const bool better = k32 < bk32;
                    bk32 = better ? k32 : bk32;
                    bidx = better ? base + 32 * k : bidx;
                }
            }
        }
        if (K16 && bk32 != 0xFFFFFFFFu) {
            const int lid = bk32 & 127;
            const uint32_t idx = Rb + (uint32_t)(w0 + lid / KS) * (uint32_t)n + (uint32_t)(lo + lane + 32 * (lid % KS));
            const uint32_t d = ((bk32 >> 7) & 0xFFFFFFu) + (uint32_t)(DELTA_BIAS - (1 << 23));
            const uint64_t key = ((uint64_t)((bk32 & 0x80000000u) | d) << 32) | idx;
            best = key < best ? key : best;
        }
    }
    if (!K16) best = bk32 == 0xFFFFFFFFu ? KEY_NONE : (((uint64_t)bk32 << 32) | bidx);
    return best;
}

// ---------------------------------------------------------------------------
// Flat tile list of one neighbourhood (used by the whole-GPU and the sharded
// kernels): relocate tiles (t-chunk, row group), swap tiles (top-aligned m2
// chunk, row group), adjacent-swap tiles (32 missions each).
struct GridTiles {
    int nTC, nSC, nAdj, nRG, G;   // t-chunks, swap chunks, adjacent tiles, row groups, rows per group
    int n_reloc, n_swap, n_total; // tile counts
    const int *swp;               // compact swap list (non-empty tiles only): swp[g] = first compact swap tile
                                  // of row group g, g = 0..nRG (a prefix over the chunk counts); null = full list
    const int *swt;               // the same list as a table g << 16 | j per compact swap tile (when it is short), or null
};

// Swap chunks j of row group g holding a pair m1 < m2 (hi = n - 64 j > m_lo + 1): the non-empty ones.
__host__ __device__ inline int swap_chunks_of_group(int n, int nSC, int G, int g) {
    const int m_lo = g * G, span = n - 1 - m_lo;
    if (span <= 0) return 0;
    const int c = (span + 32 * KS - 1) / (32 * KS);
    return c < nSC ? c : nSC;
}

__host__ __device__ inline GridTiles grid_tiles(int n, int V, int G) {
    GridTiles T;
    const int S = n + V;
    T.G = G;
    T.nTC = (S + 32 * KR - 1) / (32 * KR);
    T.nSC = n > 1 ? (n - 1 + 32 * KS - 1) / (32 * KS) : 0;
    T.nRG = (n + G - 1) / G;
    T.nAdj = (n + 31) / 32;
    T.n_reloc = T.nTC * T.nRG;
    T.n_swap = T.nSC * T.nRG;
    T.n_total = T.n_reloc + T.n_swap + T.nAdj;
    T.swp = nullptr;
    T.swt = nullptr;
    return T;
}

// The same list without the swap tiles that lie entirely on or below the diagonal (every row of the group
// at or above the chunk's top): the whole-GPU kernel's tile list on one GPU (fewer, more even tiles per warp).
__host__ __device__ inline int compact_swap_count(int n, int V, int G) {
    const GridTiles T = grid_tiles(n, V, G);
    int c = 0;
    for (int g = 0; g < T.nRG; g++) c += swap_chunks_of_group(n, T.nSC, G, g);
    return c;
}

// The FAST relocate scorer's removal side of row m (score_reloc_fast): {route a, removal delta rem}, or
// {-1, 0} when m is unassigned, the link p -> s it leaves breaks con7/con8, or route a would stay over the
// flight limit (reading #42: then no relocate of m is feasible).  Depends only on m's route.
template <class TT>
__device__ __forceinline__ int2 reloc_row_record(const TT *Ts, const int4 *CS4, const int4 *RS4, const uint32_t *LK,
                                                 const uint32_t *VC, const int32_t *F, int NL, int NLp, int P, int m) {
    const int4 rm = RS4[m];
    const int a = (int16_t)((uint32_t)rm.w >> 16);
    if (a < 0) return make_int2(-1, 0);
    const int s = LK[m] & 0xFFFF;
    const int4 rsx = RS4[s];
    const int4 csx = CS4[s];
    const int ca = VC[a] & 0xFF;
    const int Dps = (int)Ts[(ca * NL + (rm.w & 0xFFFF)) * NLp + (csx.y & 0xFFFF)] + rsx.z;
    if (rm.x + Dps > csx.x) return make_int2(-1, 0);
    const int rem = Dps - rm.y - rsx.y;
    if (F[a] + rem > P) return make_int2(-1, 0);
    return make_int2(a, rem);
}

// No-wait variant (f3) tiles: every move by the engine's exact evaluation (engine.cuh reloc_eval /
// swap_eval with NW), m warp-uniform, lanes over the targets t of the chunk / the m2 of the swap chunk
// (m2 > m1, adjacent pairs included: swap_eval is exact for them, so no adjacent-pair tiles are needed).
template <bool TABU, class TT, class ET, class MV, class RV>
__device__ __forceinline__ uint64_t score_reloc_nw(const ScoreCtx<TT, ET> &SC, const MV &M, const RV &R, int t0,
                                                   int m_lo, int m_hi, int it, long long cur, long long best,
                                                   int lane) {
    uint64_t kb = KEY_NONE;
    for (int m = m_lo; m < m_hi; m++) {
        const RelocRow r = reloc_row(M, R, m);
        if (r.a < 0) continue;
#pragma unroll
        for (int k = 0; k < KR; k++) {
            const int t = t0 + lane + 32 * k;
            if (t >= SC.S) continue;
            const MoveEval e = reloc_eval<true>(M, R, r, m, t, SC.mask, it);
            const int cls = move_class<TABU>(e, cur, best);
            if (cls >= 0) {
                const uint64_t key = make_key(cls, e.delta, (uint32_t)m * (uint32_t)SC.S + (uint32_t)t);
                kb = key < kb ? key : kb;
            }
        }
    }
    return kb;
}

template <bool TABU, class TT, class ET, class MV, class RV>
__device__ __forceinline__ uint64_t score_swap_nw(const ScoreCtx<TT, ET> &SC, const MV &M, const RV &R, int hi,
                                                  int m1_lo, int m1_hi, int it, long long cur, long long best,
                                                  int lane) {
    uint64_t kb = KEY_NONE;
    for (int m1 = m1_lo; m1 < m1_hi; m1++) {
#pragma unroll
        for (int k = 0; k < KS; k++) {
            const int m2 = hi - 32 * KS + lane + 32 * k;
            if (m2 <= m1) continue;
            const MoveEval e = swap_eval<true>(M, R, m1, m2, SC.mask, it);
            const int cls = move_class<TABU>(e, cur, best);
            if (cls >= 0) {
                const uint64_t key = make_key(cls, e.delta, SC.Rb + (uint32_t)m1 * (uint32_t)SC.n + (uint32_t)m2);
                kb = key < kb ? key : kb;
            }
        }
    }
    return kb;
}

// One tile of the flat tile list: this lane's best packed key in it.
template <bool TABU, bool FULL, bool TR, bool NW = false, class TT, class ET, class MV, class RV>
__device__ __forceinline__ uint64_t score_tile(const ScoreCtx<TT, ET> &SC, const MV &M, const RV &R,
                                               const GridTiles &GT, int tile, int it, long long cur, long long best,
                                               int lane) {
    const int n = SC.n;
    const int asp = (int)(best - cur);
    uint64_t kb = KEY_NONE;
    {
        if (tile < GT.n_reloc) {
            const int c = tile % GT.nTC, g = tile / GT.nTC;
            const int m_lo = g * GT.G, m_hi = min(n, m_lo + GT.G);
            if constexpr (NW) kb = score_reloc_nw<TABU>(SC, M, R, c * 32 * KR, m_lo, m_hi, it, cur, best, lane);
            else kb = FULL ? score_reloc_fast<TABU, TR>(SC, c * 32 * KR, m_lo, m_hi, it, asp, lane)
                           : score_reloc<TABU, FULL, TR>(SC, c * 32 * KR, m_lo, m_hi, it, asp, lane);
        } else if (tile < GT.n_reloc + GT.n_swap) {
            const int r = tile - GT.n_reloc;
            int j, g;
            if (GT.swt) {   // compact list, short: direct table
                const int e = GT.swt[r];
                g = e >> 16;
                j = e & 0xFFFF;
            } else if (GT.swp) {   // compact list: the row group by binary search over the prefix, then the chunk
                int lo_g = 0, hi_g = GT.nRG;   // swp[lo_g] <= r < swp[hi_g]
                while (hi_g - lo_g > 1) {
                    const int mid = (lo_g + hi_g) >> 1;
                    if (GT.swp[mid] <= r) lo_g = mid; else hi_g = mid;
                }
                g = lo_g;
                j = r - GT.swp[g];
            } else {
                j = r % GT.nSC;
                g = r / GT.nSC;
            }
            const int hi = n - j * 32 * KS;
            const int m_lo = g * GT.G, m_hi = min(hi - 1, m_lo + GT.G);
            if (m_lo < m_hi) {
                if constexpr (NW) kb = score_swap_nw<TABU>(SC, M, R, hi, m_lo, m_hi, it, cur, best, lane);
                else kb = FULL ? score_swap_fast<TABU, TR>(SC, hi, m_lo, m_hi, it, asp, lane)
                               : score_swap<TABU, FULL, TR>(SC, hi, m_lo, m_hi, it, asp, lane);
            }
        } else if (!NW) {
            const int x = (tile - GT.n_reloc - GT.n_swap) * 32 + lane;
            if (x < n && (FULL || (SC.mask & 8u))) {
                const int gg = SC.LK[x] & 0xFFFF;
                if (R.veh[x] >= 0 && gg < n) {
                    const int m1 = min(x, gg), m2 = max(x, gg);
                    const MoveEval e = swap_eval(M, R, m1, m2, SC.mask, it);
                    const int cls = move_class<TABU>(e, cur, best);
                    if (cls >= 0) kb = make_key(cls, e.delta, SC.Rb + (uint32_t)m1 * (uint32_t)n + (uint32_t)m2);
                }
            }
        }
    }
    return kb;
}

// Score tiles [tlo, thi) of the flat tile list with stride over the warps of the grid.
template <bool TABU, bool FULL, bool TR, bool NW = false, class TT, class ET, class MV, class RV>
__device__ __forceinline__ uint64_t score_tiles(const ScoreCtx<TT, ET> &SC, const MV &M, const RV &R,
                                                const GridTiles &GT, int tlo, int thi, int gwarp, int nwarps_all,
                                                int it, long long cur, long long best, int lane) {
    uint64_t kmin = KEY_NONE;
    for (int tile = tlo + gwarp; tile < thi; tile += nwarps_all) {
        const uint64_t kb = score_tile<TABU, FULL, TR, NW>(SC, M, R, GT, tile, it, cur, best, lane);
        kmin = kb < kmin ? kb : kmin;
    }
    return kmin;
}

}  // namespace airsched
