// engine.cuh -- device-side data layout and the per-move arithmetic of the
// move-evaluation engine (sm_100a).  Integer seconds throughout; every value
// here is exact int32/int64 arithmetic, so the GPU and the CPU oracle agree
// bit for bit.
//
// Notation follows the paper (§3-§4): mission n has pickup/delivery
// locations, deadline w_n, helicopter flag rho; a vehicle
// (base) flies base -> missions -> same base; d_{ijl} is the node
// travel time of layer l = b_k (Eq. obj_s).
//
// Slot numbering: slots 0..n-1 are missions, slot n+v is
// vehicle v's terminal: as a predecessor it is START_v (clock 0, ends at the
// base), as a successor it is END_v (deadline = day length, svc 0).  The route
// of v is a doubly linked list: succ[n+v] = first mission (or n+v when empty),
// pred[n+v] = last mission.
//
// The views are templates over the element types so the same arithmetic
// serves the wide layout (int32 everywhere: k_search, k_eval_dump) and the
// compact layout of the batched kernel (uint16 links/locations, uint16 travel
// times when they fit, int16 tabu expiries when they fit).
#pragma once
#include <cstdint>

namespace airsched {

constexpr uint64_t KEY_NONE = 0xFFFFFFFFFFFFFFFFull;
// Never a selection key (its delta field would be 2^30 - 1; |delta| < 2^29, reading #32):
// the fused sharded exchange returns it when a peer's key did not arrive in time.
constexpr uint64_t KEY_ABORT = 0x7FFFFFFFFFFFFFFFull;
constexpr int32_t DELTA_BIAS = 1 << 30;

// Instance, device-resident (uploaded once per ctx).
struct DevInst {
    const int32_t *T;        // [NC][NL][NL]
    const int32_t *vloc;     // [V] base location of vehicle v
    const int32_t *vcls;     // [V] class (matrix layer)
    const uint8_t *vcls8;    // [V] same, bytes
    const uint8_t *cls_heli; // [NC]
    const int32_t *pick;     // [n]
    const int32_t *del;      // [n]
    const int32_t *w;        // [n]
    const uint8_t *heli;     // [n]
    const int32_t *svc;      // [NC][n] = T_c[pick][del] (pickup->delivery leg)
    int32_t n, V, NL, NC, P, DAY;
    int32_t no_wait;         // f3 variant: depart on arrival (reading #40)
    int32_t maxT;            // max travel time (selects the uint16 table)
    int32_t svcpos;          // every pickup->delivery leg > 0 in every class (enables the FAST scorers)
    int32_t tsym;            // every layer of T is symmetric (the transposed table is T itself)
    const void *TpadT;       // padded table transposed per layer (== the padded table when tsym)
    const uint16_t *TDg;     // node costs TD[c][x][t] = T_c[x][pick_t] + svc_c(t) (END slots: T_c[x][base]),
                             // rows of n + V, uint16, in global memory for the global-table scorers; or null
};

// Selection key (O9): class bit 63, biased delta bits 62..32, index bits 31..0.
__host__ __device__ __forceinline__ uint64_t make_key(int cls, int32_t delta, uint32_t idx) {
    return ((uint64_t)cls << 63) | ((uint64_t)(uint32_t)(delta + DELTA_BIAS) << 32) | (uint64_t)idx;
}
__host__ __device__ __forceinline__ int key_cls(uint64_t k) { return (int)(k >> 63); }
__host__ __device__ __forceinline__ int32_t key_delta(uint64_t k) {
    return (int32_t)((uint32_t)(k >> 32) & 0x7FFFFFFFu) - DELTA_BIAS;
}
__host__ __device__ __forceinline__ uint32_t key_idx(uint64_t k) { return (uint32_t)k; }

// Read-only per-instance constants as seen by the kernels (smem or global).
// Engine code reads them through the accessors cls/hok/vl/dl/hl/sv so other
// layouts (the batched kernel's AoS records) can provide the same interface.
template <class LocT, class TT>
struct MissionViewT {
    const TT *T;            // [NC][NL][NLp]
    const LocT *del;        // [n]
    const uint8_t *heli;    // [n] 0/1
    const int32_t *svc;     // [NC][n]
    const uint8_t *vcls;    // [V]
    const LocT *vloc;       // [V]
    const uint8_t *clsheli; // [NC]
    int32_t n, V, NL, NLp, P, DAY;
    __device__ __forceinline__ int cls(int v) const { return vcls[v]; }
    __device__ __forceinline__ int hok(int c) const { return clsheli[c]; }
    __device__ __forceinline__ int vl(int v) const { return (int)vloc[v]; }
    __device__ __forceinline__ int dl(int m) const { return (int)del[m]; }
    __device__ __forceinline__ int hl(int m) const { return heli[m]; }
    __device__ __forceinline__ int sv(int c, int m) const { return svc[c * n + m]; }
};

// Strided field of an array-of-structs record in (shared) memory: lets the
// engine's R.field[x] syntax address AoS layouts.
template <class T, int STRIDE, int OFF>
struct Field {
    unsigned char *base;
    __device__ __forceinline__ T &operator[](int x) const {
        return *reinterpret_cast<T *>(base + x * STRIDE + OFF);
    }
};

// Mutable per-run state.
template <class VehT, class LinkT, class LocT, class ET>
struct RunViewT {
    LinkT *succ, *pred;             // [S] linked lists
    VehT *veh;                      // [S] vehicle of a slot; -1 if unassigned
    LocT *endc;                     // [S] end location of the predecessor
    int32_t *depc, *inc;            // [S] predecessor's departure (w_pred, 0 at START); d(pred, slot)
    int32_t *svco;                  // [S] own pickup->delivery leg in the slot's class (0 for END)
    const LocT *pick_s;             // [S] pickup (base location for END)
    const int32_t *w_s;             // [S] deadline (day length for END)
    int32_t *F;                     // [V] route flight time (con6)
    ET *E;                          // [n][V] tabu expiry (nullable)
    // no-wait variant only (f3; null otherwise).  depc then holds the
    // predecessor's ARRIVAL (its departure when it does not wait).
    int32_t *arr;                   // [S] arrival at the slot (END: return to base)
    int32_t *sl;                    // [S] min over the route suffix from the slot of (w - arr)
    int32_t *pos;                   // [S] position in the route (missions 1..L, END L+1)
    int32_t *slp;                   // [S] first position of the suffix where that minimum is attained
};

using MissionView = MissionViewT<int32_t, int32_t>;
using RunView = RunViewT<int32_t, int32_t, int32_t, int32_t>;

template <class MV>
__device__ __forceinline__ int32_t Tget(const MV &M, int c, int a, int b) {
    return (int32_t)M.T[(c * M.NL + a) * M.NLp + b];
}

// Recompute the incoming-link record of slot x from pred[x] (apply / init).
template <class MV, class RV>
__device__ __forceinline__ void refresh_slot(const MV &M, const RV &R, int x) {
    const int n = M.n;
    int p = R.pred[x];
    int v = x < n ? (int)R.veh[x] : x - n;
    int c = M.cls(v);
    int e = p < n ? M.dl(p) : M.vl(p - n);
    int d = p < n ? R.w_s[p] : 0;
    int sv = x < n ? M.sv(c, x) : 0;
    R.endc[x] = e;
    R.depc[x] = d;
    R.svco[x] = sv;
    R.inc[x] = Tget(M, c, e, R.pick_s[x]) + sv;
}

// ---- relocate (O5 relocate block): remove m, insert before slot t ---------
// Per-row (m-uniform) part: the removal side, amortised over the t loop.
struct RelocRow {
    int a, s, ca;             // route of m, successor slot, class of a
    int rem;                  // d(p,s) - d(p,m) - d(m,s)
    int Dps;                  // d(p,s)
    bool rem_ok;              // dep(p) + d(p,s) <= w(s)
    int pick_m, del_m, w_m, heli_m;
    int Fa;
};

template <class MV, class RV>
__device__ __forceinline__ RelocRow reloc_row(const MV &M, const RV &R, int m) {
    RelocRow r;
    r.a = R.veh[m];
    if (r.a < 0) return r;
    r.s = R.succ[m];
    r.ca = M.cls(r.a);
    int Dps = Tget(M, r.ca, R.endc[m], R.pick_s[r.s]) + R.svco[r.s];
    r.rem = Dps - R.inc[m] - R.inc[r.s];
    r.Dps = Dps;
    r.rem_ok = R.depc[m] + Dps <= R.w_s[r.s];
    r.pick_m = R.pick_s[m];
    r.del_m = M.dl(m);
    r.w_m = R.w_s[m];
    r.heli_m = M.hl(m);
    r.Fa = R.F[r.a];
    return r;
}

struct MoveEval {
    bool valid, feasible, tabu;
    int32_t delta;
    int32_t da, db;     // per-route flight deltas (db unused when same route)
};

__device__ __forceinline__ MoveEval move_none() {
    MoveEval e;
    e.valid = e.feasible = e.tabu = false;
    e.delta = e.da = e.db = 0;
    return e;
}

// ---- no-wait variant (f3, reading #40) ---------------------------
// Without waiting a route's clock carries arrivals, so a move shifts every
// later arrival of the route by the same amount: the route stays feasible iff
// each shifted stretch keeps its slack.  min(w - arr) over the stretch x..y
// (inclusive, along succ):
template <class RV>
__device__ __forceinline__ int nw_range_slack(const RV &R, int x, int y) {
    int s = 0x7FFFFFFF;
    for (;;) {
        int v = R.w_s[x] - R.arr[x];
        s = v < s ? v : s;
        if (x == y) break;
        x = R.succ[x];
    }
    return s;
}

// Does every slot of the stretch x..y (x at or before y along succ) keep slack >= d?
// O(1) unless the suffix minimum from x is below d and lies after y: then the
// stretch's own minimum decides (walk).  Same answer as d <= nw_range_slack.
template <class RV>
__device__ __forceinline__ bool nw_stretch_ok(const RV &R, int x, int y, int d) {
    if (d <= R.sl[x]) return true;                 // the whole suffix from x has the slack
    if (R.slp[x] <= R.pos[y]) return false;        // its minimum (< d) lies inside x..y
    return d <= nw_range_slack(R, x, y);
}

// Recompute the whole route of vehicle v (incoming-link records, arrivals,
// positions, suffix slacks and where they are attained) from its linked list.
// Single thread, O(L).
template <class MV, class RV>
__device__ inline void nw_refresh_route(const MV &M, const RV &R, int v) {
    const int n = M.n, term = n + v, c = M.cls(v);
    int e = M.vl(v), dep = 0, k = 0;
    int x = R.succ[term];
    for (;;) {
        int sv = x < n ? M.sv(c, x) : 0;
        int inc = Tget(M, c, e, R.pick_s[x]) + sv;
        R.endc[x] = e;
        R.depc[x] = dep;
        R.svco[x] = sv;
        R.inc[x] = inc;
        R.arr[x] = dep + inc;
        R.pos[x] = ++k;
        if (x >= n) break;
        e = M.dl(x);
        dep += inc;
        x = R.succ[x];
    }
    int s = 0x7FFFFFFF, sp = 0;
    x = term;
    do {
        int v2 = R.w_s[x] - R.arr[x];
        if (v2 <= s) { s = v2; sp = R.pos[x]; }   // ties: the earlier position
        R.sl[x] = s;
        R.slp[x] = sp;
        x = R.pred[x];
    } while (x != term);
}

// Time feasibility of relocating m (route a: p -> m -> s) before t (route b,
// c = pred t); x1 = d(c, m), x2 = d(m, t) in b's class.
template <class MV, class RV>
__device__ __forceinline__ bool nw_reloc_time(const MV &M, const RV &R, const RelocRow &r, int m, int t, int b,
                                              int x1, int x2) {
    const int s = r.s;
    if (b != r.a) {
        if (R.depc[m] + r.Dps - R.arr[s] > R.sl[s]) return false;        // a: s.. shifted
        int Am = R.depc[t] + x1;                                           // b: c -> m -> t..
        return Am <= r.w_m && Am + x2 - R.arr[t] <= R.sl[t];
    }
    if (R.pos[t] > R.pos[m]) {               // p s .. c m t ..
        int c = R.pred[t];
        int d1 = R.depc[m] + r.Dps - R.arr[s];
        if (!nw_stretch_ok(R, s, c, d1)) return false;
        int Am = R.arr[c] + d1 + x1;
        return Am <= r.w_m && Am + x2 - R.arr[t] <= R.sl[t];
    }
    const int p = R.pred[m];                 // c m t .. p s ..
    int Am = R.depc[t] + x1;
    if (Am > r.w_m) return false;
    int d1 = Am + x2 - R.arr[t];
    if (!nw_stretch_ok(R, t, p, d1)) return false;
    return R.arr[p] + d1 + r.Dps - R.arr[s] <= R.sl[s];
}

// Insert part for target slot t (t != m, t != succ(m), both assigned).
template <bool NW = false, class MV, class RV>
__device__ __forceinline__ MoveEval reloc_eval(const MV &M, const RV &R, const RelocRow &r, int m, int t,
                                                uint32_t mask, int it) {
    MoveEval e = move_none();
    if (r.a < 0 || t == m || t == r.s) return e;
    int b = R.veh[t];
    if (b < 0) return e;
    if (!(mask & (b != r.a ? 1u : 2u))) return e;
    e.valid = true;
    int cb = M.cls(b);
    int x1 = Tget(M, cb, R.endc[t], r.pick_m) + M.sv(cb, m);   // d(c, m)
    int x2 = Tget(M, cb, r.del_m, R.pick_s[t]) + R.svco[t];             // d(m, t)
    int ins = x1 + x2 - R.inc[t];
    e.delta = r.rem + ins;
    bool ok = !r.heli_m || M.hok(cb);
    if constexpr (NW) ok = ok && nw_reloc_time(M, R, r, m, t, b, x1, x2);
    else ok = ok && r.rem_ok && (R.depc[t] + x1 <= r.w_m) && (r.w_m + x2 <= R.w_s[t]);
    if (b == r.a) {
        ok = ok && (r.Fa + e.delta <= M.P);
        e.da = e.delta;
    } else {
        ok = ok && (r.Fa + r.rem <= M.P) && (R.F[b] + ins <= M.P);
        e.da = r.rem;
        e.db = ins;
    }
    e.feasible = ok;
    if (R.E) e.tabu = (int)R.E[m * M.V + b] >= it;
    return e;
}

// ---- swap (O5 swap block): exchange the positions of m1 < m2 --------------
template <bool NW = false, class MV, class RV>
__device__ __forceinline__ MoveEval swap_eval(const MV &M, const RV &R, int m1, int m2, uint32_t mask, int it) {
    MoveEval e = move_none();
    int a = R.veh[m1], b = R.veh[m2];
    if (a < 0 || b < 0) return e;
    if (!(mask & (a != b ? 4u : 8u))) return e;
    e.valid = true;
    const int n = M.n;
    int s1 = R.succ[m1], s2 = R.succ[m2];
    int ca = M.cls(a);
    int pick1 = R.pick_s[m1], pick2 = R.pick_s[m2];
    int del1 = M.dl(m1), del2 = M.dl(m2);
    int w1 = R.w_s[m1], w2 = R.w_s[m2];
    int Fa = R.F[a];
    if (s1 == m2 || s2 == m1) {
        // adjacent in one route: p -> f -> g -> s becomes p -> g -> f -> s
        int f = s1 == m2 ? m1 : m2;   // first of the pair in the route
        int g = s1 == m2 ? m2 : m1;   // second
        int sg = s1 == m2 ? s2 : s1;  // successor of the pair
        int delf = f == m1 ? del1 : del2, delg = g == m1 ? del1 : del2;
        int pickf = f == m1 ? pick1 : pick2, pickg = g == m1 ? pick1 : pick2;
        int wf = f == m1 ? w1 : w2, wg = g == m1 ? w1 : w2;
        int y1 = Tget(M, ca, R.endc[f], pickg) + M.sv(ca, g);      // p -> g
        int y2 = Tget(M, ca, delg, pickf) + M.sv(ca, f);           // g -> f
        int y3 = Tget(M, ca, delf, R.pick_s[sg]) + R.svco[sg];           // f -> s
        e.delta = y1 + y2 + y3 - R.inc[f] - R.inc[g] - R.inc[sg];
        e.da = e.delta;
        if constexpr (NW) {
            int Ag = R.depc[f] + y1, Af = Ag + y2;   // no waiting: arrivals chain
            e.feasible = (Ag <= wg) && (Af <= wf) && (Af + y3 - R.arr[sg] <= R.sl[sg]) && (Fa + e.delta <= M.P);
        } else {
            e.feasible = (R.depc[f] + y1 <= wg) && (wg + y2 <= wf) && (wf + y3 <= R.w_s[sg]) && (Fa + e.delta <= M.P);
        }
    } else {
        int cb = M.cls(b);
        int ya1 = Tget(M, ca, R.endc[m1], pick2) + M.sv(ca, m2);   // p1 -> m2
        int ya2 = Tget(M, ca, del2, R.pick_s[s1]) + R.svco[s1];          // m2 -> s1
        int yb1 = Tget(M, cb, R.endc[m2], pick1) + M.sv(cb, m1);   // p2 -> m1
        int yb2 = Tget(M, cb, del1, R.pick_s[s2]) + R.svco[s2];          // m1 -> s2
        e.da = ya1 + ya2 - R.inc[m1] - R.inc[s1];
        e.db = yb1 + yb2 - R.inc[m2] - R.inc[s2];
        e.delta = e.da + e.db;
        bool ok = (!M.hl(m2) || M.hok(ca)) && (!M.hl(m1) || M.hok(cb));
        if constexpr (NW) {
            if (a != b) {
                int A2 = R.depc[m1] + ya1, A1 = R.depc[m2] + yb1;
                ok = ok && (A2 <= w2) && (A2 + ya2 - R.arr[s1] <= R.sl[s1]) && (A1 <= w1) &&
                     (A1 + yb2 - R.arr[s2] <= R.sl[s2]);
            } else {
                // one route, not adjacent: pf f sf .. pg g sg -> pf g sf .. pg f sg
                const bool first1 = R.pos[m1] < R.pos[m2];
                const int f = first1 ? m1 : m2, g = first1 ? m2 : m1;
                const int sf = first1 ? s1 : s2, sg = first1 ? s2 : s1, pg = R.pred[g];
                const int d_pf_g = first1 ? ya1 : yb1, d_g_sf = first1 ? ya2 : yb2;
                const int d_pg_f = first1 ? yb1 : ya1, d_f_sg = first1 ? yb2 : ya2;
                const int wf = first1 ? w1 : w2, wg = first1 ? w2 : w1;
                int Ag = R.depc[f] + d_pf_g;
                int d1 = Ag + d_g_sf - R.arr[sf];
                ok = ok && (Ag <= wg) && nw_stretch_ok(R, sf, pg, d1);
                int Af = R.arr[pg] + d1 + d_pg_f;
                ok = ok && (Af <= wf) && (Af + d_f_sg - R.arr[sg] <= R.sl[sg]);
            }
        } else {
            ok = ok && (R.depc[m1] + ya1 <= w2) && (w2 + ya2 <= R.w_s[s1]) && (R.depc[m2] + yb1 <= w1) &&
                 (w1 + yb2 <= R.w_s[s2]);
        }
        if (a == b) ok = ok && (Fa + e.delta <= M.P);
        else ok = ok && (Fa + e.da <= M.P) && (R.F[b] + e.db <= M.P);
        e.feasible = ok;
    }
    if (R.E) e.tabu = ((int)R.E[m1 * M.V + b] >= it) || ((int)R.E[m2 * M.V + a] >= it);
    return e;
}

// Selection class (O9): 0 admissible, 1 by-default, -1 not selectable.
template <bool TABU>
__device__ __forceinline__ int move_class(const MoveEval &e, long long cur, long long best) {
    if (!e.valid || !e.feasible) return -1;
    bool adm = TABU ? (!e.tabu || cur + (long long)e.delta < best) : (e.delta < 0);
    return adm ? 0 : 1;
}

// Evaluate canonical index idx (decode + score); used by the dump kernel and apply.
template <bool NW = false, class MV, class RV>
__device__ __forceinline__ MoveEval eval_index(const MV &M, const RV &R, uint32_t idx, uint32_t mask, int it) {
    const int n = M.n, S = M.n + M.V;
    uint32_t Rb = (uint32_t)n * (uint32_t)S;
    if (idx < Rb) {
        int m = idx / S, t = idx % S;
        RelocRow r = reloc_row(M, R, m);
        if (r.a < 0) return move_none();
        return reloc_eval<NW>(M, R, r, m, t, mask, it);
    }
    uint32_t k = idx - Rb;
    int m1 = k / n, m2 = k % n;
    if (m1 >= m2) return move_none();
    return swap_eval<NW>(M, R, m1, m2, mask, it);
}

// Per-route split of a VALID move's delta (read BEFORE the move is applied):
// a, b = the routes of m (m1) and t (m2); da, db = their flight-time changes
// (db = 0 when a == b).  The scorers already proved validity and feasibility, so
// only the removal side (relocate) or route a's two new links (swap) are needed.
struct MoveSplit {
    int a, b;
    int32_t da, db;
};

template <class MV, class RV>
__device__ __forceinline__ MoveSplit move_split(const MV &M, const RV &R, uint32_t idx, int32_t delta) {
    const int n = M.n, S = M.n + M.V;
    const uint32_t Rb = (uint32_t)n * (uint32_t)S;
    MoveSplit r;
    if (idx < Rb) {
        const int m = idx / S, t = idx % S;
        r.a = R.veh[m];
        r.b = R.veh[t];
        if (r.a == r.b) { r.da = delta; r.db = 0; return r; }
        const int s = R.succ[m];
        const int Dps = Tget(M, M.cls(r.a), R.endc[m], R.pick_s[s]) + R.svco[s];
        r.da = Dps - R.inc[m] - R.inc[s];
        r.db = delta - r.da;
        return r;
    }
    const uint32_t k = idx - Rb;
    const int m1 = k / n, m2 = k % n;
    r.a = R.veh[m1];
    r.b = R.veh[m2];
    const int s1 = R.succ[m1];
    if (r.a == r.b) { r.da = delta; r.db = 0; return r; }   // (adjacent pairs share a route)
    const int ca = M.cls(r.a);
    const int ya1 = Tget(M, ca, R.endc[m1], R.pick_s[m2]) + M.sv(ca, m2);
    const int ya2 = Tget(M, ca, M.dl(m2), R.pick_s[s1]) + R.svco[s1];
    r.da = ya1 + ya2 - R.inc[m1] - R.inc[s1];
    r.db = delta - r.da;
    return r;
}

// Relink the lists for a VALID move (pre-move routes a, b from move_split) and
// list the slots whose incoming-link record must be refreshed (<= 4).  Route
// totals and records are the caller's.
template <class MV, class RV>
__device__ __forceinline__ int move_relink(const MV &M, const RV &R, uint32_t idx, int a, int b, int *touched) {
    const int n = M.n, S = M.n + M.V;
    const uint32_t Rb = (uint32_t)n * (uint32_t)S;
    if (idx < Rb) {
        const int m = idx / S, t = idx % S;
        const int p = R.pred[m], s = R.succ[m];
        const int c = R.pred[t];   // t's predecessor after the removal too: a valid t is neither m nor succ(m)
        R.succ[p] = s;
        R.pred[s] = p;
        R.succ[c] = m;
        R.pred[m] = c;
        R.succ[m] = t;
        R.pred[t] = m;
        R.veh[m] = b;
        touched[0] = s; touched[1] = m; touched[2] = t;
        return 3;
    }
    const uint32_t k = idx - Rb;
    const int m1 = k / n, m2 = k % n;
    const int p1 = R.pred[m1], s1 = R.succ[m1], p2 = R.pred[m2], s2 = R.succ[m2];
    if (s1 == m2) {          // p1 m1 m2 s2 -> p1 m2 m1 s2
        R.succ[p1] = m2; R.pred[m2] = p1; R.succ[m2] = m1; R.pred[m1] = m2; R.succ[m1] = s2; R.pred[s2] = m1;
        touched[0] = m2; touched[1] = m1; touched[2] = s2;
        return 3;
    }
    if (s2 == m1) {          // p2 m2 m1 s1 -> p2 m1 m2 s1
        R.succ[p2] = m1; R.pred[m1] = p2; R.succ[m1] = m2; R.pred[m2] = m1; R.succ[m2] = s1; R.pred[s1] = m2;
        touched[0] = m1; touched[1] = m2; touched[2] = s1;
        return 3;
    }
    R.succ[p1] = m2; R.pred[m2] = p1; R.succ[m2] = s1; R.pred[s1] = m2;
    R.succ[p2] = m1; R.pred[m1] = p2; R.succ[m1] = s2; R.pred[s2] = m1;
    R.veh[m1] = b;
    R.veh[m2] = a;
    touched[0] = m1; touched[1] = m2; touched[2] = s1; touched[3] = s2;
    return 4;
}

// Route totals (con6) and the tabu expiry of the 'from' pairs (O8) after a move.
template <class MV, class RV>
__device__ __forceinline__ void move_totals(const MV &M, const RV &R, uint32_t idx, const MoveSplit &ms, int it,
                                            int tenure, bool write_tabu) {
    R.F[ms.a] += ms.da;
    if (ms.b != ms.a) R.F[ms.b] += ms.db;
    if (!(write_tabu && R.E)) return;
    const int n = M.n, S = M.n + M.V;
    const uint32_t Rb = (uint32_t)n * (uint32_t)S;
    if (idx < Rb) {
        R.E[(idx / S) * M.V + ms.a] = it + tenure;
    } else {
        const uint32_t k = idx - Rb;
        R.E[(k / n) * M.V + ms.a] = it + tenure;
        R.E[(k % n) * M.V + ms.b] = it + tenure;
    }
}

// Apply a VALID move whose delta is e.delta (single thread): split, relink,
// refresh the touched incoming-link records (no-wait: recompute the touched
// routes), route totals, tabu expiries.
template <bool NW = false, class MV, class RV>
__device__ inline void apply_move(const MV &M, const RV &R, uint32_t idx, const MoveEval &e, int it, int tenure,
                                  bool write_tabu) {
    const MoveSplit ms = move_split(M, R, idx, e.delta);
    int touched[4];
    const int nt = move_relink(M, R, idx, ms.a, ms.b, touched);
    if constexpr (NW) {
        nw_refresh_route(M, R, ms.a);
        if (ms.b != ms.a) nw_refresh_route(M, R, ms.b);
    } else {
        for (int q = 0; q < nt; q++) refresh_slot(M, R, touched[q]);
    }
    move_totals(M, R, idx, ms, it, tenure, write_tabu);
}

__host__ __device__ __forceinline__ uint64_t splitmix64_next(uint64_t &s) {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// FNV-1a-64 of the tabu list in force after iteration it (O8): triples
// (m, v, E[m][v]) with E >= it+1, (m, v) order, little-endian int32 bytes.
template <class ET>
__device__ inline uint64_t tabu_digest(const ET *E, int n, int V, int it) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int mm = 0; mm < n; mm++)
        for (int v = 0; v < V; v++) {
            int ev = E[mm * V + v];
            if (ev < it + 1) continue;
            int trip[3] = {mm, v, ev};
            for (int q3 = 0; q3 < 3; q3++)
                for (int by = 0; by < 4; by++) {
                    h ^= (uint64_t)(((uint32_t)trip[q3] >> (8 * by)) & 0xFFu);
                    h *= 0x100000001b3ull;
                }
        }
    return h;
}

}  // namespace airsched
