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
// Slot numbering: slots 0..n-1 are missions, slot
// n+v is vehicle v's terminal: as a predecessor it is START_v (clock 0, ends
// at the base), as a successor it is END_v (deadline = day length, svc 0).
// The route of v is a doubly linked list: succ[n+v] = first mission (or n+v
// when empty), pred[n+v] = last mission.
#pragma once
#include <cstdint>

namespace airsched {

constexpr uint64_t KEY_NONE = 0xFFFFFFFFFFFFFFFFull;
constexpr int32_t DELTA_BIAS = 1 << 30;

// Instance, device-resident (uploaded once per ctx).
struct DevInst {
    const int32_t *T;        // [NC][NL][NL]
    const int32_t *vloc;     // [V] base location of vehicle v
    const int32_t *vcls;     // [V] class (matrix layer)
    const uint8_t *cls_heli; // [NC]
    const int32_t *pick;     // [n]
    const int32_t *del;      // [n]
    const int32_t *w;        // [n]
    const uint8_t *heli;     // [n]
    const int32_t *svc;      // [NC][n] = T_c[pick][del] (pickup->delivery leg)
    int32_t n, V, NL, NC, P, DAY;
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

// Mutable per-run state.  All pointers refer to one run (shared memory in
// the persistent kernels, global memory in the dump kernel).
struct RunView {
    int32_t *succ, *pred, *veh;     // [S] linked lists; veh[m] = -1 if unassigned
    int32_t *endc, *depc, *inc;     // [S] per-slot record of the incoming link:
                                    //   endc = end location of pred, depc = departure
                                    //   time of pred (w_pred, 0 at START), inc = d(pred, slot)
    int32_t *svco;                  // [S] own pickup->delivery leg in the slot's class (0 for END)
    const int32_t *pick_s, *w_s;    // [S] pickup (base for END) and deadline (DAY for END)
    int32_t *F;                     // [V] route flight time (con6)
    int32_t *E;                     // [n][V] tabu expiry (nullable)
};

// Read-only per-mission constants as seen by the kernels (may be staged in smem).
struct MissionView {
    const int32_t *del;   // [n]
    const int32_t *heli;  // [n] 0/1
    const int32_t *svc;   // [NC][n]
    const int32_t *vcls;  // [V]
    const int32_t *vloc;  // [V]
    const int32_t *clsheli; // [NC]
    const int32_t *T;     // [NC][NL][NL] (smem or global)
    int32_t n, V, NL, P, DAY;
};

__device__ __forceinline__ int32_t Tget(const MissionView &M, int c, int a, int b) {
    return M.T[(c * M.NL + a) * M.NL + b];
}

// Recompute the incoming-link record of slot x from pred[x] (apply / init).
__device__ __forceinline__ void refresh_slot(const MissionView &M, const RunView &R, int x) {
    const int n = M.n;
    int p = R.pred[x];
    int v = x < n ? R.veh[x] : x - n;
    int c = M.vcls[v];
    int e = p < n ? M.del[p] : M.vloc[p - n];
    int d = p < n ? R.w_s[p] : 0;
    int sv = x < n ? M.svc[c * n + x] : 0;
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
    bool rem_ok;              // dep(p) + d(p,s) <= w(s)
    int pick_m, del_m, w_m, heli_m;
    int Fa;
};

__device__ __forceinline__ RelocRow reloc_row(const MissionView &M, const RunView &R, int m) {
    RelocRow r;
    r.a = R.veh[m];
    if (r.a < 0) return r;
    r.s = R.succ[m];
    r.ca = M.vcls[r.a];
    int Dps = Tget(M, r.ca, R.endc[m], R.pick_s[r.s]) + R.svco[r.s];
    r.rem = Dps - R.inc[m] - R.inc[r.s];
    r.rem_ok = R.depc[m] + Dps <= R.w_s[r.s];
    r.pick_m = R.pick_s[m];
    r.del_m = M.del[m];
    r.w_m = R.w_s[m];
    r.heli_m = M.heli[m];
    r.Fa = R.F[r.a];
    return r;
}

struct MoveEval {
    bool valid, feasible, tabu;
    int32_t delta;
    int32_t da, db;     // per-route flight deltas (db unused when same route)
};

// Insert part for target slot t (t != m, t != succ(m), both assigned).
__device__ __forceinline__ MoveEval reloc_eval(const MissionView &M, const RunView &R, const RelocRow &r, int m,
                                                int t, uint32_t mask, int it) {
    MoveEval e;
    e.valid = false;
    e.feasible = false;
    e.tabu = false;
    e.delta = 0;
    e.da = e.db = 0;
    if (r.a < 0 || t == m || t == r.s) return e;
    int b = R.veh[t];
    if (b < 0) return e;
    if (!(mask & (b != r.a ? 1u : 2u))) return e;
    e.valid = true;
    int cb = M.vcls[b];
    int x1 = Tget(M, cb, R.endc[t], r.pick_m) + M.svc[cb * M.n + m];   // d(c, m)
    int x2 = Tget(M, cb, r.del_m, R.pick_s[t]) + R.svco[t];             // d(m, t)
    int ins = x1 + x2 - R.inc[t];
    e.delta = r.rem + ins;
    bool ok = r.rem_ok && (!r.heli_m || M.clsheli[cb]) && (R.depc[t] + x1 <= r.w_m) && (r.w_m + x2 <= R.w_s[t]);
    if (b == r.a) {
        ok = ok && (r.Fa + e.delta <= M.P);
        e.da = e.delta;
    } else {
        ok = ok && (r.Fa + r.rem <= M.P) && (R.F[b] + ins <= M.P);
        e.da = r.rem;
        e.db = ins;
    }
    e.feasible = ok;
    if (R.E) e.tabu = R.E[m * M.V + b] >= it;
    return e;
}

// ---- swap (O5 swap block): exchange the positions of m1 < m2 --------------
__device__ __forceinline__ MoveEval swap_eval(const MissionView &M, const RunView &R, int m1, int m2, uint32_t mask,
                                              int it) {
    MoveEval e;
    e.valid = false;
    e.feasible = false;
    e.tabu = false;
    e.delta = 0;
    e.da = e.db = 0;
    int a = R.veh[m1], b = R.veh[m2];
    if (a < 0 || b < 0) return e;
    if (!(mask & (a != b ? 4u : 8u))) return e;
    e.valid = true;
    const int n = M.n;
    int s1 = R.succ[m1], s2 = R.succ[m2];
    int ca = M.vcls[a];
    int pick1 = R.pick_s[m1], pick2 = R.pick_s[m2];
    int del1 = M.del[m1], del2 = M.del[m2];
    int w1 = R.w_s[m1], w2 = R.w_s[m2];
    int Fa = R.F[a];
    if (s1 == m2 || s2 == m1) {
        // adjacent: x -> y -> z becomes x -> z' ... with (first, second) = order in route
        int f = s1 == m2 ? m1 : m2;   // first of the pair in the route
        int g = s1 == m2 ? m2 : m1;   // second
        int sg = s1 == m2 ? s2 : s1;  // successor of the pair
        int delf = f == m1 ? del1 : del2, delg = g == m1 ? del1 : del2;
        int pickf = f == m1 ? pick1 : pick2, pickg = g == m1 ? pick1 : pick2;
        int wf = f == m1 ? w1 : w2, wg = g == m1 ? w1 : w2;
        int y1 = Tget(M, ca, R.endc[f], pickg) + M.svc[ca * n + g];      // p -> g
        int y2 = Tget(M, ca, delg, pickf) + M.svc[ca * n + f];           // g -> f
        int y3 = Tget(M, ca, delf, R.pick_s[sg]) + R.svco[sg];           // f -> s
        e.delta = y1 + y2 + y3 - R.inc[f] - R.inc[g] - R.inc[sg];
        e.da = e.delta;
        e.feasible = (R.depc[f] + y1 <= wg) && (wg + y2 <= wf) && (wf + y3 <= R.w_s[sg]) && (Fa + e.delta <= M.P);
    } else {
        int cb = M.vcls[b];
        int ya1 = Tget(M, ca, R.endc[m1], pick2) + M.svc[ca * n + m2];   // p1 -> m2
        int ya2 = Tget(M, ca, del2, R.pick_s[s1]) + R.svco[s1];          // m2 -> s1
        int yb1 = Tget(M, cb, R.endc[m2], pick1) + M.svc[cb * n + m1];   // p2 -> m1
        int yb2 = Tget(M, cb, del1, R.pick_s[s2]) + R.svco[s2];          // m1 -> s2
        e.da = ya1 + ya2 - R.inc[m1] - R.inc[s1];
        e.db = yb1 + yb2 - R.inc[m2] - R.inc[s2];
        e.delta = e.da + e.db;
        bool ok = (!M.heli[m2] || M.clsheli[ca]) && (!M.heli[m1] || M.clsheli[cb]) &&
                  (R.depc[m1] + ya1 <= w2) && (w2 + ya2 <= R.w_s[s1]) && (R.depc[m2] + yb1 <= w1) &&
                  (w1 + yb2 <= R.w_s[s2]);
        if (a == b) ok = ok && (Fa + e.delta <= M.P);
        else ok = ok && (Fa + e.da <= M.P) && (R.F[b] + e.db <= M.P);
        e.feasible = ok;
    }
    if (R.E) e.tabu = (R.E[m1 * M.V + b] >= it) || (R.E[m2 * M.V + a] >= it);
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
__device__ __forceinline__ MoveEval eval_index(const MissionView &M, const RunView &R, uint32_t idx, uint32_t mask,
                                               int it) {
    const int n = M.n, S = M.n + M.V;
    uint32_t Rb = (uint32_t)n * (uint32_t)S;
    if (idx < Rb) {
        int m = idx / S, t = idx % S;
        RelocRow r = reloc_row(M, R, m);
        if (r.a < 0) {
            MoveEval e;
            e.valid = e.feasible = e.tabu = false;
            e.delta = e.da = e.db = 0;
            return e;
        }
        return reloc_eval(M, R, r, m, t, mask, it);
    }
    uint32_t k = idx - Rb;
    int m1 = k / n, m2 = k % n;
    if (m1 >= m2) {
        MoveEval e;
        e.valid = e.feasible = e.tabu = false;
        e.delta = e.da = e.db = 0;
        return e;
    }
    return swap_eval(M, R, m1, m2, mask, it);
}

// Apply a VALID move whose per-route deltas are in e (single thread).
// Relinks the lists, refreshes the incoming-link records of the touched slots,
// updates route flight totals and the tabu expiry of the 'from' pairs (O8).
__device__ inline void apply_move(const MissionView &M, const RunView &R, uint32_t idx, const MoveEval &e, int it,
                                  int tenure, bool write_tabu) {
    const int n = M.n, S = M.n + M.V;
    uint32_t Rb = (uint32_t)n * (uint32_t)S;
    if (idx < Rb) {
        int m = idx / S, t = idx % S;
        int a = R.veh[m];
        int b = R.veh[t];
        int p = R.pred[m], s = R.succ[m];
        R.succ[p] = s;
        R.pred[s] = p;
        int c = R.pred[t];
        R.succ[c] = m;
        R.pred[m] = c;
        R.succ[m] = t;
        R.pred[t] = m;
        R.veh[m] = b;
        refresh_slot(M, R, s);
        refresh_slot(M, R, m);
        refresh_slot(M, R, t);
        if (a == b) R.F[a] += e.delta;
        else { R.F[a] += e.da; R.F[b] += e.db; }
        if (write_tabu && R.E) R.E[m * M.V + a] = it + tenure;
    } else {
        uint32_t k = idx - Rb;
        int m1 = k / n, m2 = k % n;
        int a = R.veh[m1], b = R.veh[m2];
        int p1 = R.pred[m1], s1 = R.succ[m1], p2 = R.pred[m2], s2 = R.succ[m2];
        if (s1 == m2) {          // p1 m1 m2 s2 -> p1 m2 m1 s2
            R.succ[p1] = m2; R.pred[m2] = p1; R.succ[m2] = m1; R.pred[m1] = m2; R.succ[m1] = s2; R.pred[s2] = m1;
            refresh_slot(M, R, m2); refresh_slot(M, R, m1); refresh_slot(M, R, s2);
            R.F[a] += e.delta;
        } else if (s2 == m1) {   // p2 m2 m1 s1 -> p2 m1 m2 s1
            R.succ[p2] = m1; R.pred[m1] = p2; R.succ[m1] = m2; R.pred[m2] = m1; R.succ[m2] = s1; R.pred[s1] = m2;
            refresh_slot(M, R, m1); refresh_slot(M, R, m2); refresh_slot(M, R, s1);
            R.F[a] += e.delta;
        } else {
            R.succ[p1] = m2; R.pred[m2] = p1; R.succ[m2] = s1; R.pred[s1] = m2;
            R.succ[p2] = m1; R.pred[m1] = p2; R.succ[m1] = s2; R.pred[s2] = m1;
            R.veh[m1] = b;
            R.veh[m2] = a;
            refresh_slot(M, R, m1); refresh_slot(M, R, m2); refresh_slot(M, R, s1); refresh_slot(M, R, s2);
            if (a == b) R.F[a] += e.delta;
            else { R.F[a] += e.da; R.F[b] += e.db; }
        }
        if (write_tabu && R.E) {
            R.E[m1 * M.V + a] = it + tenure;
            R.E[m2 * M.V + b] = it + tenure;
        }
    }
}

__host__ __device__ __forceinline__ uint64_t splitmix64_next(uint64_t &s) {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace airsched
