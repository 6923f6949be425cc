/*
 * oracle.c -- CPU ORACLE for arXiv 2002.11710's neighbourhood / tabu search.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain, slow, obviously correct:
 * no incremental deltas, no linked lists, no packed keys.  Every move is
 * applied to copies of the routes it touches and the routes are re-costed
 * and re-checked from the definitions.  Section / line citations refer to
 * /root/reference/PAPER.md ("P:n"); readings #k refer to DESIGN.md's
 * ambiguity ledger (= SURVEY.md §8(c).2).
 */
#define _POSIX_C_SOURCE 200809L  /* pthread barriers (the parallel driver) */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- O1/O2 -- */
/* Node travel time d_{ijl} (reading #1): arriving at a mission
 * node means flying from the end of the previous node to the pickup and then
 * from the pickup to the delivery point.  A base node ends at the base. */
static int32_t T_at(const or_inst *I, int32_t c, int32_t a, int32_t b) {
    return I->T[((int64_t)c * I->NL + a) * I->NL + b];
}

/* end location of route element x: x >= 0 is mission x (ends at its delivery
 * point), x < 0 is the vehicle's base (START/END). */
static int32_t end_loc(const or_inst *I, int32_t v, int32_t x) {
    return x >= 0 ? I->del[x] : I->veh_loc[v];
}

/* D_c(x, y) for y a mission */
static int64_t D_to_mission(const or_inst *I, int32_t v, int32_t x, int32_t y) {
    int32_t c = I->veh_cls[v];
    return (int64_t)T_at(I, c, end_loc(I, v, x), I->pick[y]) + T_at(I, c, I->pick[y], I->del[y]);
}

/* D_c(x, END_v) */
static int64_t D_to_base(const or_inst *I, int32_t v, int32_t x) {
    int32_t c = I->veh_cls[v];
    return T_at(I, c, end_loc(I, v, x), I->veh_loc[v]);
}

/* ------------------------------------------------------------------- O3 -- */
/* Eq. obj_s: sum of x_ijk d_ijl over the links of route v, l = b_k.
 * Empty route: cost 0 ("none at all"; reading #10). */
int64_t or_route_cost(const or_inst *I, int32_t v, const int32_t *route, int32_t L) {
    if (L == 0) return 0;
    int64_t cost = 0;
    int32_t prev = -1; /* START_v */
    for (int32_t i = 0; i < L; i++) {
        cost += D_to_mission(I, v, prev, route[i]);
        prev = route[i];
    }
    cost += D_to_base(I, v, prev);
    return cost;
}

/* ------------------------------------------------------------------- O4 -- */
/* (f3, reading #40: with no_wait the vehicle departs a mission on arrival, so
 * the clock carries the arrival time instead of the deadline; deadlines stay
 * upper bounds on arrival.)
 * Route feasibility:
 *  (i)  con7/con8 (text P:148; readings #2-#6): the clock starts
 *       at 0 at the base, the vehicle departs mission x at exactly w_x, and
 *       every arrival is <= the next deadline; the return arrives by DAY
 *       (reading #7);
 *  (ii) con6: flight time (waiting excluded) <= p;
 *  (iii) con9 (reading #9): no helicopter-only mission on a plane. */
int32_t or_route_feasible(const or_inst *I, int32_t v, const int32_t *route, int32_t L) {
    if (L == 0) return 1;
    int64_t dep = 0;
    int32_t prev = -1;
    for (int32_t i = 0; i < L; i++) {
        int32_t m = route[i];
        if (I->heli[m] && !I->class_is_heli[I->veh_cls[v]]) return 0;
        int64_t arrival = dep + D_to_mission(I, v, prev, m);
        if (arrival > I->w[m]) return 0;
        dep = I->no_wait ? arrival : I->w[m];
        prev = m;
    }
    if (dep + D_to_base(I, v, prev) > I->DAY) return 0;
    if (or_route_cost(I, v, route, L) > I->P) return 0;
    return 1;
}

int64_t or_objective(const or_inst *I, const int32_t *len, const int32_t *r) {
    int64_t s = 0;
    for (int32_t v = 0; v < I->V; v++) s += or_route_cost(I, v, r + (int64_t)v * I->n, len[v]);
    return s;
}

/* con1/con2: every mission served exactly once; plus O4 per route. */
int32_t or_schedule_feasible(const or_inst *I, const int32_t *len, const int32_t *r) {
    int32_t n = I->n;
    int32_t *seen = (int32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
    int32_t ok = 1;
    for (int32_t v = 0; v < I->V && ok; v++) {
        for (int32_t i = 0; i < len[v]; i++) {
            int32_t m = r[(int64_t)v * n + i];
            if (m < 0 || m >= n || seen[m]) { ok = 0; break; }
            seen[m] = 1;
        }
        if (ok && !or_route_feasible(I, v, r + (int64_t)v * n, len[v])) ok = 0;
    }
    for (int32_t m = 0; m < n && ok; m++)
        if (!seen[m]) ok = 0;
    free(seen);
    return ok;
}

/* ------------------------------------------------------------------- O5 -- */
int64_t or_move_space_size(const or_inst *I) {
    int64_t n = I->n, V = I->V;
    return n * (n + V) + n * n;
}

/* where each mission sits; veh = -1 if unassigned (partial schedules, O13) */
static void locate(const or_inst *I, const int32_t *len, const int32_t *r, int32_t *veh, int32_t *pos) {
    for (int32_t m = 0; m < I->n; m++) { veh[m] = -1; pos[m] = -1; }
    for (int32_t v = 0; v < I->V; v++)
        for (int32_t i = 0; i < len[v]; i++) {
            int32_t m = r[(int64_t)v * I->n + i];
            veh[m] = v;
            pos[m] = i;
        }
}

static void remove_at(int32_t *route, int32_t *L, int32_t i) {
    for (int32_t k = i; k + 1 < *L; k++) route[k] = route[k + 1];
    (*L)--;
}

static void insert_at(int32_t *route, int32_t *L, int32_t i, int32_t m) {
    for (int32_t k = *L; k > i; k--) route[k] = route[k - 1];
    route[i] = m;
    (*L)++;
}

static int32_t index_of(const int32_t *route, int32_t L, int32_t m) {
    for (int32_t i = 0; i < L; i++)
        if (route[i] == m) return i;
    return -1;
}

/* Decode move idx and build the affected routes (copies).
 *   relocate block idx = m*(n+V) + t : remove m, insert it immediately before
 *     mission t (as the routes stand after the removal) or, for t >= n, at the
 *     end of route t-n.  VALID iff m and t are assigned, t != m and t is not
 *     m's successor slot (those two are no-ops).  Inter-route relocate is the
 *     paper's move (Alg. 2, Fig. 2); intra-route reorder and swap
 *     are BASELINE.json north_star's extensions (reading #13).
 *   swap block idx = n(n+V) + m1*n + m2 : exchange the positions of m1 and m2;
 *     VALID iff m1 < m2, both assigned.
 * mask bits: 1 inter-relocate, 2 intra-relocate, 4 inter-swap, 8 intra-swap.
 * Outputs: a, b (b == a when one route), new routes ra[0..*la) and rb[0..*lb).
 * Also the (mission, vehicle) pairs a move places into a vehicle (O7). */
typedef struct {
    int32_t a, b;
    int32_t la, lb;
    int32_t into_m[2], into_v[2], from_m[2], from_v[2], n_pairs;
} move_t;

static int32_t build_move(const or_inst *I, const int32_t *len, const int32_t *r, const int32_t *veh,
                          const int32_t *pos, int64_t idx, uint32_t mask, move_t *mv, int32_t *ra,
                          int32_t *rb) {
    int64_t n = I->n, V = I->V;
    if (idx < 0 || idx >= or_move_space_size(I)) return 0;
    if (idx < n * (n + V)) {
        int32_t m = (int32_t)(idx / (n + V));
        int32_t t = (int32_t)(idx % (n + V));
        if (veh[m] < 0) return 0;
        int32_t a = veh[m];
        int32_t La = len[a];
        int32_t succslot = pos[m] + 1 < La ? r[(int64_t)a * n + pos[m] + 1] : (int32_t)(n + a);
        if (t == m || t == succslot) return 0;
        int32_t b;
        if (t < n) {
            if (veh[t] < 0) return 0;
            b = veh[t];
        } else {
            b = t - (int32_t)n;
        }
        if (!(mask & (a != b ? 1u : 2u))) return 0;
        mv->a = a;
        mv->b = b;
        memcpy(ra, r + (int64_t)a * n, sizeof(int32_t) * (size_t)La);
        mv->la = La;
        remove_at(ra, &mv->la, pos[m]);
        if (a == b) {
            int32_t at = t < n ? index_of(ra, mv->la, t) : mv->la;
            insert_at(ra, &mv->la, at, m);
            mv->lb = 0;
        } else {
            int32_t Lb = len[b];
            memcpy(rb, r + (int64_t)b * n, sizeof(int32_t) * (size_t)Lb);
            mv->lb = Lb;
            int32_t at = t < n ? index_of(rb, Lb, t) : Lb;
            insert_at(rb, &mv->lb, at, m);
        }
        mv->n_pairs = 1;
        mv->into_m[0] = m; mv->into_v[0] = b;
        mv->from_m[0] = m; mv->from_v[0] = a;
        return 1;
    } else {
        int64_t k = idx - n * (n + V);
        int32_t m1 = (int32_t)(k / n), m2 = (int32_t)(k % n);
        if (!(m1 < m2)) return 0;
        if (veh[m1] < 0 || veh[m2] < 0) return 0;
        int32_t a = veh[m1], b = veh[m2];
        if (!(mask & (a != b ? 4u : 8u))) return 0;
        mv->a = a;
        mv->b = b;
        memcpy(ra, r + (int64_t)a * n, sizeof(int32_t) * (size_t)len[a]);
        mv->la = len[a];
        if (a == b) {
            ra[pos[m1]] = m2;
            ra[pos[m2]] = m1;
            mv->lb = 0;
        } else {
            memcpy(rb, r + (int64_t)b * n, sizeof(int32_t) * (size_t)len[b]);
            mv->lb = len[b];
            ra[pos[m1]] = m2;
            rb[pos[m2]] = m1;
        }
        mv->n_pairs = 2;
        mv->into_m[0] = m1; mv->into_v[0] = b;
        mv->into_m[1] = m2; mv->into_v[1] = a;
        mv->from_m[0] = m1; mv->from_v[0] = a;
        mv->from_m[1] = m2; mv->from_v[1] = b;
        return 1;
    }
}

static void write_back(const or_inst *I, int32_t *len, int32_t *r, const move_t *mv, const int32_t *ra,
                       const int32_t *rb) {
    int64_t n = I->n;
    memcpy(r + (int64_t)mv->a * n, ra, sizeof(int32_t) * (size_t)mv->la);
    len[mv->a] = mv->la;
    if (mv->b != mv->a) {
        memcpy(r + (int64_t)mv->b * n, rb, sizeof(int32_t) * (size_t)mv->lb);
        len[mv->b] = mv->lb;
    }
}

int32_t or_apply_move(const or_inst *I, const int32_t *len, const int32_t *r, int64_t idx, uint32_t mask,
                      int32_t *len_out, int32_t *r_out) {
    int32_t n = I->n, V = I->V;
    int32_t *veh = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *ra = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *rb = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    locate(I, len, r, veh, pos);
    move_t mv;
    int32_t ok = build_move(I, len, r, veh, pos, idx, mask, &mv, ra, rb);
    memcpy(len_out, len, sizeof(int32_t) * (size_t)V);
    memcpy(r_out, r, sizeof(int32_t) * (size_t)V * (size_t)n);
    if (ok) write_back(I, len_out, r_out, &mv, ra, rb);
    free(veh); free(pos); free(ra); free(rb);
    return ok;
}

/* ------------------------------------------------------------- O6-O9 ---- */
typedef struct {
    const or_inst *I;
    int32_t *veh, *pos, *ra, *rb, *len_full, *r_full;
    int64_t *route_cost;
    int64_t cur;
} evalctx;

static void evalctx_init(evalctx *X, const or_inst *I, const int32_t *len, const int32_t *r) {
    int32_t n = I->n, V = I->V;
    X->I = I;
    X->veh = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    X->pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    X->ra = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    X->rb = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    X->len_full = (int32_t *)malloc(sizeof(int32_t) * (size_t)V);
    X->r_full = (int32_t *)malloc(sizeof(int32_t) * (size_t)V * (size_t)(n + 1));
    X->route_cost = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    locate(I, len, r, X->veh, X->pos);
    X->cur = 0;
    for (int32_t v = 0; v < V; v++) {
        X->route_cost[v] = or_route_cost(I, v, r + (int64_t)v * n, len[v]);
        X->cur += X->route_cost[v];
    }
}

static void evalctx_free(evalctx *X) {
    free(X->veh); free(X->pos); free(X->ra); free(X->rb);
    free(X->len_full); free(X->r_full); free(X->route_cost);
}

/* Delta and feasibility of one move: Delta = Obj(apply(S,mv)) - Obj(S) (O6),
 * FEASIBLE = O4 of the new routes (route-local) or of the whole new schedule
 * (full).  Returns VALID. */
static int32_t eval_one(evalctx *X, const int32_t *len, const int32_t *r, int64_t idx, uint32_t mask,
                        int32_t full, move_t *mv, int64_t *delta, int32_t *feasible) {
    const or_inst *I = X->I;
    if (!build_move(I, len, r, X->veh, X->pos, idx, mask, mv, X->ra, X->rb)) return 0;
    if (full) {
        memcpy(X->len_full, len, sizeof(int32_t) * (size_t)I->V);
        memcpy(X->r_full, r, sizeof(int32_t) * (size_t)I->V * (size_t)I->n);
        write_back(I, X->len_full, X->r_full, mv, X->ra, X->rb);
        *delta = or_objective(I, X->len_full, X->r_full) - or_objective(I, len, r);
        int32_t ok = 1;
        for (int32_t v = 0; v < I->V && ok; v++)
            ok = or_route_feasible(I, v, X->r_full + (int64_t)v * I->n, X->len_full[v]);
        *feasible = ok;
        return 1;
    }
    int64_t before = X->route_cost[mv->a] + (mv->b != mv->a ? X->route_cost[mv->b] : 0);
    int64_t after = or_route_cost(I, mv->a, X->ra, mv->la);
    int32_t ok = or_route_feasible(I, mv->a, X->ra, mv->la);
    if (mv->b != mv->a) {
        after += or_route_cost(I, mv->b, X->rb, mv->lb);
        ok = ok && or_route_feasible(I, mv->b, X->rb, mv->lb);
    }
    *delta = after - before;
    *feasible = ok;
    return 1;
}

/* O7/O8: a move is TABU iff some (mission, vehicle) pair it places into has
 * E[m][v] >= it (TabuList/TabuCounter, Alg. 3; readings
 * #18, #20). */
static int32_t is_tabu(const or_inst *I, const move_t *mv, const int32_t *E, int32_t it) {
    if (!E) return 0;
    for (int32_t k = 0; k < mv->n_pairs; k++)
        if (E[(int64_t)mv->into_m[k] * I->V + mv->into_v[k]] >= it) return 1;
    return 0;
}

/* O9 selection over all indices, ascending, strict "better" => the lowest
 * index wins ties (CurrentMin; reading #26).  TS: ADMISSIBLE =
 * FEASIBLE and (not TABU or cur+Delta < best) (aspiration, reading #21).
 * NS: ADMISSIBLE = FEASIBLE and Delta < 0 (reading #17).  If nothing is
 * admissible, the best FEASIBLE move is the by-default choice (class 1). */
static void select_move(evalctx *X, const int32_t *len, const int32_t *r, int32_t mode, const int32_t *E,
                        int32_t it, int64_t best_obj, uint32_t mask, int32_t full, int32_t *delta_out,
                        uint8_t *flags_out, int32_t *best_cls, int64_t *best_delta, int64_t *best_idx) {
    const or_inst *I = X->I;
    int64_t N = or_move_space_size(I);
    int64_t adm_idx = -1, adm_delta = 0, def_idx = -1, def_delta = 0;
    for (int64_t idx = 0; idx < N; idx++) {
        move_t mv;
        int64_t delta = 0;
        int32_t feas = 0;
        uint8_t flags = 0;
        if (eval_one(X, len, r, idx, mask, full, &mv, &delta, &feas)) {
            flags |= OR_FLAG_VALID;
            int32_t admissible = 0;
            if (feas) flags |= OR_FLAG_FEASIBLE;
            if (mode == OR_MODE_TABU) {
                int32_t tabu = is_tabu(I, &mv, E, it);
                if (tabu) flags |= OR_FLAG_TABU;
                admissible = feas && (!tabu || X->cur + delta < best_obj);
            } else {
                admissible = feas && delta < 0;
            }
            if (admissible) {
                flags |= OR_FLAG_ADMISSIBLE;
                if (adm_idx < 0 || delta < adm_delta) { adm_idx = idx; adm_delta = delta; }
            } else if (feas) {
                flags |= OR_FLAG_BYDEFAULT;
                if (def_idx < 0 || delta < def_delta) { def_idx = idx; def_delta = delta; }
            }
        }
        if (delta_out) delta_out[idx] = (int32_t)delta;
        if (flags_out) flags_out[idx] = flags;
    }
    if (adm_idx >= 0) { *best_cls = 0; *best_delta = adm_delta; *best_idx = adm_idx; }
    else if (def_idx >= 0) { *best_cls = 1; *best_delta = def_delta; *best_idx = def_idx; }
    else { *best_cls = -1; *best_delta = 0; *best_idx = -1; }
}

void or_eval_moves(const or_inst *I, const int32_t *len, const int32_t *r, int32_t mode, const int32_t *E,
                   int32_t it, int64_t best_obj, uint32_t mask, int32_t full, int32_t *delta_out,
                   uint8_t *flags_out, int32_t *best_cls, int32_t *best_delta, int64_t *best_idx) {
    evalctx X;
    evalctx_init(&X, I, len, r);
    int64_t bd = 0;
    select_move(&X, len, r, mode, E, it, best_obj, mask, full, delta_out, flags_out, best_cls, &bd, best_idx);
    *best_delta = (int32_t)bd;
    evalctx_free(&X);
}

/* The same per-index values for a list of indices (large instances, sampled). */
void or_eval_index_list(const or_inst *I, const int32_t *len, const int32_t *r, int32_t mode, const int32_t *E,
                        int32_t it, int64_t best_obj, uint32_t mask, int64_t count, const int64_t *idx,
                        int32_t *delta_out, uint8_t *flags_out) {
    evalctx X;
    evalctx_init(&X, I, len, r);
    for (int64_t k = 0; k < count; k++) {
        move_t mv;
        int64_t delta = 0;
        int32_t feas = 0;
        uint8_t flags = 0;
        if (eval_one(&X, len, r, idx[k], mask, 0, &mv, &delta, &feas)) {
            int32_t admissible;
            flags |= OR_FLAG_VALID;
            if (feas) flags |= OR_FLAG_FEASIBLE;
            if (mode == OR_MODE_TABU) {
                int32_t tabu = is_tabu(I, &mv, E, it);
                if (tabu) flags |= OR_FLAG_TABU;
                admissible = feas && (!tabu || X.cur + delta < best_obj);
            } else {
                admissible = feas && delta < 0;
            }
            if (admissible) flags |= OR_FLAG_ADMISSIBLE;
            else if (feas) flags |= OR_FLAG_BYDEFAULT;
        }
        delta_out[k] = (int32_t)delta;
        flags_out[k] = flags;
    }
    evalctx_free(&X);
}

/* ------------------------------------------------------------------ O12 -- */
/* SplitMix64 (Steele, Lea & Flood 2014) -- the run seed's generator. */
uint64_t or_splitmix64_next(uint64_t *state) {
    *state += 0x9E3779B97F4A7C15ull;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Seeded kick: for k < kick, draw up to 64 relocate indices z mod n(n+V) and
 * apply the first VALID and FEASIBLE one (all move kinds enabled; no tabu
 * entries, no iteration advance).  seed 0 = no kick (reading #27). */
int32_t or_kick(const or_inst *I, int32_t *len, int32_t *r, uint64_t seed, int32_t kick) {
    if (seed == 0 || I->n == 0) return 0;
    uint64_t s = seed;
    int64_t R = (int64_t)I->n * (I->n + I->V);
    int32_t applied = 0;
    for (int32_t k = 0; k < kick; k++) {
        for (int32_t tries = 0; tries < 64; tries++) {
            int64_t idx = (int64_t)(or_splitmix64_next(&s) % (uint64_t)R);
            evalctx X;
            evalctx_init(&X, I, len, r);
            move_t mv;
            int64_t delta;
            int32_t feas;
            int32_t valid = eval_one(&X, len, r, idx, 0xFu, 0, &mv, &delta, &feas);
            if (valid && feas) write_back(I, len, r, &mv, X.ra, X.rb);
            evalctx_free(&X);
            if (valid && feas) { applied++; break; }
        }
    }
    return applied;
}

/* ------------------------------------------------------------------ O8 --- */
/* FNV-1a-64 over the little-endian bytes of the int32 triples (m, v, E[m][v])
 * with E >= it+1, in (m, v) order: the tabu list in force after iteration it. */
uint64_t or_tabu_digest(const or_inst *I, const int32_t *E, int32_t it) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int32_t m = 0; m < I->n; m++)
        for (int32_t v = 0; v < I->V; v++) {
            int32_t e = E[(int64_t)m * I->V + v];
            if (e < it + 1) continue;
            int32_t trip[3] = {m, v, e};
            for (int32_t q = 0; q < 3; q++)
                for (int32_t byte = 0; byte < 4; byte++) {
                    h ^= (uint64_t)(((uint32_t)trip[q] >> (8 * byte)) & 0xFFu);
                    h *= 0x100000001b3ull;
                }
        }
    return h;
}

/* ------------------------------------------------------------ O10/O11 ---- */
/* Alg. 2 / Alg. 3 in north_star's global-best form (reading #16): one
 * iteration = evaluate the whole neighbourhood, apply the selected move. */
int32_t or_search(const or_inst *I, const int32_t *len0, const int32_t *r0, const or_params *prm,
                  int32_t *best_len, int32_t *best_r, int32_t *final_len, int32_t *final_r, or_result *res,
                  int64_t *tr_idx, int32_t *tr_delta, int64_t *tr_cur, int64_t *tr_best, int32_t *tr_cls,
                  uint64_t *tr_digest, int32_t *E_out) {
    int32_t n = I->n, V = I->V;
    size_t rs = sizeof(int32_t) * (size_t)V * (size_t)(n > 0 ? n : 1);
    int32_t *len = (int32_t *)malloc(sizeof(int32_t) * (size_t)V);
    int32_t *r = (int32_t *)malloc(rs);
    int32_t *E = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1) * (size_t)V);
    memcpy(len, len0, sizeof(int32_t) * (size_t)V);
    memcpy(r, r0, rs);
    for (int64_t k = 0; k < (int64_t)n * V; k++) E[k] = -1;  /* O8: initialised to -1 */

    memset(res, 0, sizeof(*res));
    res->kicks_applied = or_kick(I, len, r, prm->seed, prm->kick);
    int64_t cur = or_objective(I, len, r);
    int64_t best = cur;
    res->start_obj = cur;
    res->best_iter = -1;
    res->stop_reason = 0; /* MAX_ITERS */
    memcpy(best_len, len, sizeof(int32_t) * (size_t)V);
    memcpy(best_r, r, rs);
    int32_t it;
    for (it = 0; it < prm->max_iters; it++) {
        evalctx X;
        evalctx_init(&X, I, len, r);
        int32_t cls;
        int64_t delta, idx;
        select_move(&X, len, r, prm->mode, prm->mode == OR_MODE_TABU ? E : NULL, it, best, prm->mask, 0,
                    NULL, NULL, &cls, &delta, &idx);
        if (cls < 0) { evalctx_free(&X); res->stop_reason = 2; break; }     /* NO_FEASIBLE_MOVE */
        if (cls == 1 && prm->mode == OR_MODE_NS) { evalctx_free(&X); res->stop_reason = 1; break; } /* LOCAL_OPT */
        if (cls == 1 && prm->strict_tabu_stop) { evalctx_free(&X); res->stop_reason = 2; break; }  /* ALL_TABU */
        move_t mv;
        int64_t d2;
        int32_t f2;
        eval_one(&X, len, r, idx, prm->mask, 0, &mv, &d2, &f2);
        write_back(I, len, r, &mv, X.ra, X.rb);
        evalctx_free(&X);
        cur += delta;
        if (prm->mode == OR_MODE_TABU)       /* O8: E[from pairs] = it + tenure */
            for (int32_t k = 0; k < mv.n_pairs; k++)
                E[(int64_t)mv.from_m[k] * V + mv.from_v[k]] = it + prm->tenure;
        if (cur < best) {
            best = cur;
            res->best_iter = it;
            memcpy(best_len, len, sizeof(int32_t) * (size_t)V);
            memcpy(best_r, r, rs);
        }
        if (tr_idx) tr_idx[it] = idx;
        if (tr_delta) tr_delta[it] = (int32_t)delta;
        if (tr_cur) tr_cur[it] = cur;
        if (tr_best) tr_best[it] = best;
        if (tr_cls) tr_cls[it] = cls;
        if (tr_digest && prm->want_digest) tr_digest[it] = or_tabu_digest(I, E, it);
    }
    res->iters_done = it;
    res->best_obj = best;
    res->final_obj = cur;
    if (final_len) memcpy(final_len, len, sizeof(int32_t) * (size_t)V);
    if (final_r) memcpy(final_r, r, rs);
    if (E_out) memcpy(E_out, E, sizeof(int32_t) * (size_t)n * (size_t)V);
    free(len); free(r); free(E);
    return 0;
}

/* ------------------------------------------------------------------ O13 -- */
/* Algorithm 1.  Phase 1: helicopter-only missions;
 * phase 2: the rest; each by ascending (deadline, id) (line 8 "smallest
 * value in MissionTimes").  Every vehicle is scanned in id order
 * (line 7); the candidate position is the route tail (reading #23; TAIL) or
 * the deadline-sorted slot (SORTED, "placed between two indicies");
 * the candidate must keep the route feasible (lines 10-31) and CurrentMin
 * keeps the smallest cost increase, ties to the lower vehicle (P:208,
 * reading #24).  If no vehicle fits: fail if nothing is assigned yet,
 * otherwise run one NS iteration over the assigned missions ("mission swaps
 * from Algorithm 2"; "only performs a single iteration") and
 * retry the same mission once (reading #22); fail if that finds no improving
 * move, if the retry fails, or after max_repairs repairs. */
static int32_t greedy_try(const or_inst *I, int32_t insert_mode, int32_t m, const int32_t *len, const int32_t *r,
                          int32_t *best_v, int32_t *best_at, int32_t *tmp) {
    int32_t n = I->n;
    int64_t best_inc = 0;
    *best_v = -1;
    for (int32_t v = 0; v < I->V; v++) {
        const int32_t *route = r + (int64_t)v * n;
        int32_t L = len[v];
        int32_t at = L;
        if (insert_mode == 1) {
            at = 0;
            while (at < L && I->w[route[at]] <= I->w[m]) at++;
        }
        memcpy(tmp, route, sizeof(int32_t) * (size_t)L);
        int32_t L2 = L;
        insert_at(tmp, &L2, at, m);
        if (!or_route_feasible(I, v, tmp, L2)) continue;
        int64_t inc = or_route_cost(I, v, tmp, L2) - or_route_cost(I, v, route, L);
        if (*best_v < 0 || inc < best_inc) { *best_v = v; *best_at = at; best_inc = inc; }
    }
    return *best_v >= 0;
}

int32_t or_greedy(const or_inst *I, int32_t insert_mode, int32_t max_repairs, int32_t *len_out, int32_t *r_out,
                  int32_t *n_repairs, int32_t *order_out) {
    return or_greedy_seeded(I, insert_mode, max_repairs, 0, len_out, r_out, n_repairs, order_out);
}

/* f2 randomized starts (reading #41): seed != 0 replaces each phase's
 * deadline order by a permutation of it -- SplitMix64(seed) Fisher-Yates from the
 * top, phase 0 (helicopter-only) first, one generator stream, as the sweep's
 * permutation vectors.  seed 0 is Algorithm 1 as written. */
int32_t or_greedy_seeded(const or_inst *I, int32_t insert_mode, int32_t max_repairs, uint64_t seed,
                         int32_t *len_out, int32_t *r_out, int32_t *n_repairs, int32_t *order_out) {
    int32_t n = I->n, V = I->V;
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *len2 = (int32_t *)malloc(sizeof(int32_t) * (size_t)V);
    int32_t *r2 = (int32_t *)malloc(sizeof(int32_t) * (size_t)V * (size_t)(n + 1));
    /* placement order: phase (heli-only first), then deadline, then id */
    int32_t k = 0;
    for (int32_t phase = 0; phase < 2; phase++) {
        int32_t start = k;
        for (int32_t m = 0; m < n; m++)
            if ((phase == 0) == (I->heli[m] != 0)) order[k++] = m;
        for (int32_t i = start + 1; i < k; i++) {  /* insertion sort by (w, id) */
            int32_t x = order[i], j = i - 1;
            while (j >= start && (I->w[order[j]] > I->w[x] || (I->w[order[j]] == I->w[x] && order[j] > x))) {
                order[j + 1] = order[j];
                j--;
            }
            order[j + 1] = x;
        }
    }
    if (seed) {
        uint64_t st = seed;
        int32_t n0 = 0;
        for (int32_t m = 0; m < n; m++) n0 += I->heli[m] != 0;
        int32_t lo[2] = {0, n0}, hi[2] = {n0, n};
        for (int32_t ph = 0; ph < 2; ph++)
            for (int32_t x = hi[ph] - 1; x >= lo[ph] + 1; x--) {
                int32_t y = lo[ph] + (int32_t)(or_splitmix64_next(&st) % (uint64_t)(x - lo[ph] + 1));
                int32_t tmp = order[x]; order[x] = order[y]; order[y] = tmp;
            }
    }
    for (int32_t v = 0; v < V; v++) len_out[v] = 0;
    *n_repairs = 0;
    int32_t status = 0, assigned = 0;
    for (int32_t i = 0; i < n && status == 0; i++) {
        int32_t m = order[i], bv, bat;
        if (!greedy_try(I, insert_mode, m, len_out, r_out, &bv, &bat, tmp)) {
            if (assigned == 0 || *n_repairs >= max_repairs) { status = 3; break; }
            evalctx X;
            evalctx_init(&X, I, len_out, r_out);
            int32_t cls;
            int64_t delta, idx;
            select_move(&X, len_out, r_out, OR_MODE_NS, NULL, 0, 0, 0xFu, 0, NULL, NULL, &cls, &delta, &idx);
            if (cls != 0) { evalctx_free(&X); status = 3; break; }
            move_t mv;
            int64_t d2;
            int32_t f2;
            eval_one(&X, len_out, r_out, idx, 0xFu, 0, &mv, &d2, &f2);
            write_back(I, len_out, r_out, &mv, X.ra, X.rb);
            evalctx_free(&X);
            (*n_repairs)++;
            if (!greedy_try(I, insert_mode, m, len_out, r_out, &bv, &bat, tmp)) { status = 3; break; }
        }
        int32_t *route = r_out + (int64_t)bv * n;
        insert_at(route, &len_out[bv], bat, m);
        assigned++;
    }
    if (order_out) memcpy(order_out, order, sizeof(int32_t) * (size_t)n);
    free(order); free(tmp); free(len2); free(r2);
    return status;
}

/* ------------------------------------------------------- f1: Alg. 2 / 3 sweep */
/* The paper-literal sweep (reading #39): for each
 * vehicle i ("for i <- 1 to number of bases"; seeded permutation vectors,
 * P:269), for each mission j of route i as it stood when i's turn began,
 * CurrentMin = the best (delta, idx) inter-route relocate of j (k != i, P:299-301;
 * every position) that is feasible and admissible (NS: delta
 * < 0; TS: (j, k) not tabu or cur + delta < best); if CurrentMin is not
 * empty it is applied (P:331-333 / P:408-411) and, in TS, (j, i) becomes tabu for
 * `tenure` steps (expiry = step + tenure, one step per (i, j)).  NS stops
 * after a sweep without a move ("while improvement"); TS after max_steps or
 * a sweep without a move.  Permutations: SplitMix64(seed), Fisher-Yates from the
 * top, vehicles first then each route snapshot; seed 0 = identity order. */
int32_t or_sweep(const or_inst *I, const int32_t *len0, const int32_t *r0, const or_params *prm,
                 int32_t *best_len, int32_t *best_r, or_result *res, int64_t *tr_idx, int32_t *tr_delta,
                 int64_t *tr_cur, int64_t *tr_best) {
    int32_t n = I->n, V = I->V;
    size_t rs = sizeof(int32_t) * (size_t)V * (size_t)(n > 0 ? n : 1);
    int32_t *len = (int32_t *)malloc(sizeof(int32_t) * (size_t)V);
    int32_t *r = (int32_t *)malloc(rs);
    int32_t *E = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1) * (size_t)V);
    int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)V);
    int32_t *snap = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    memcpy(len, len0, sizeof(int32_t) * (size_t)V);
    memcpy(r, r0, rs);
    for (int64_t k = 0; k < (int64_t)n * V; k++) E[k] = -1;
    memset(res, 0, sizeof(*res));
    int64_t cur = or_objective(I, len, r), best = cur;
    res->start_obj = cur;
    res->best_iter = -1;
    memcpy(best_len, len, sizeof(int32_t) * (size_t)V);
    memcpy(best_r, r, rs);
    uint64_t s = prm->seed;
    int32_t step = 0, stop = 0;
    const int64_t S = (int64_t)n + V;
    while (!stop && step < prm->max_iters) {
        int32_t moved = 0;
        for (int32_t v = 0; v < V; v++) perm[v] = v;
        if (prm->seed)
            for (int32_t x = V - 1; x >= 1; x--) {
                int32_t y = (int32_t)(or_splitmix64_next(&s) % (uint64_t)(x + 1));
                int32_t tmp = perm[x]; perm[x] = perm[y]; perm[y] = tmp;
            }
        for (int32_t pi = 0; pi < V && !stop; pi++) {
            int32_t i = perm[pi];
            int32_t L = len[i];
            memcpy(snap, r + (int64_t)i * n, sizeof(int32_t) * (size_t)L);
            if (prm->seed)
                for (int32_t x = L - 1; x >= 1; x--) {
                    int32_t y = (int32_t)(or_splitmix64_next(&s) % (uint64_t)(x + 1));
                    int32_t tmp = snap[x]; snap[x] = snap[y]; snap[y] = tmp;
                }
            for (int32_t jj = 0; jj < L; jj++) {
                int32_t j = snap[jj];
                evalctx X;
                evalctx_init(&X, I, len, r);
                int64_t bidx = -1, bdelta = 0;
                for (int64_t t = 0; t < S; t++) {
                    move_t mv;
                    int64_t delta;
                    int32_t feas;
                    int64_t idx = (int64_t)j * S + t;
                    if (!eval_one(&X, len, r, idx, 1u /* inter-route relocate */, 0, &mv, &delta, &feas)) continue;
                    if (!feas) continue;
                    int32_t adm = prm->mode == OR_MODE_TABU ? (!is_tabu(I, &mv, E, step) || cur + delta < best)
                                                            : delta < 0;
                    if (adm && (bidx < 0 || delta < bdelta)) { bidx = idx; bdelta = delta; }
                }
                if (bidx >= 0) {
                    move_t mv;
                    int64_t d2;
                    int32_t f2;
                    eval_one(&X, len, r, bidx, 1u, 0, &mv, &d2, &f2);
                    write_back(I, len, r, &mv, X.ra, X.rb);
                    cur += bdelta;
                    moved = 1;
                    if (prm->mode == OR_MODE_TABU) E[(int64_t)mv.from_m[0] * V + mv.from_v[0]] = step + prm->tenure;
                    if (cur < best) {
                        best = cur;
                        res->best_iter = step;
                        memcpy(best_len, len, sizeof(int32_t) * (size_t)V);
                        memcpy(best_r, r, rs);
                    }
                }
                evalctx_free(&X);
                if (tr_idx) tr_idx[step] = bidx;
                if (tr_delta) tr_delta[step] = (int32_t)(bidx >= 0 ? bdelta : 0);
                if (tr_cur) tr_cur[step] = cur;
                if (tr_best) tr_best[step] = best;
                step++;
                if (step >= prm->max_iters) { stop = 1; break; }
            }
        }
        if (!moved && !stop) { res->stop_reason = prm->mode == OR_MODE_NS ? 1 : 2; break; }
    }
    res->iters_done = step;
    res->best_obj = best;
    res->final_obj = cur;
    free(len); free(r); free(E); free(perm); free(snap);
    return 0;
}

/* ------------------------------------------- parallel driver of O10/O11 -- */
/* A faster DRIVER of the same search for the full-length parity checks on the
 * large configs (C4: 20,000 iterations over 393,750 valid moves; C5: 1,000
 * over 24.4 M).  It changes no arithmetic: every per-move value still comes
 * from eval_one / is_tabu above, and the selection rule is select_move's
 * (admissible before by-default, smallest delta, lowest index).  Two things
 * differ, both pinned against or_search (tests/test_oracle_driver.py):
 *   (1) the canonical index range is cut into `threads` contiguous chunks
 *       scanned concurrently; each chunk keeps its lowest-index minimum with
 *       select_move's strict '<', and the chunk results are merged in chunk
 *       order with the same strict '<' -- the global lowest-index minimum;
 *   (2) with memo != 0, a move's (VALID, FEASIBLE, delta) is kept from the
 *       previous iteration unless the move touches a route the last applied
 *       move changed.  eval_one reads only the routes of the move's m (m1)
 *       and t (m2) (route-local mode), and a mission changes route only if it
 *       lies in a changed route before and after, so a move whose routes are
 *       both unchanged has the same values; TABU and ADMISSIBLE depend on E,
 *       it, cur and best and are recomputed for every move every iteration. */
#include <pthread.h>

typedef struct {
    const or_inst *I;
    const int32_t *len, *r;
    const or_params *prm;
    const int32_t *E;
    int32_t it;
    int64_t best_obj, lo, hi;
    int32_t memo, first;
    const uint8_t *changed;    /* [V] routes changed by the last move */
    int32_t *m_delta;          /* memo [N] */
    uint8_t *m_flags;          /* memo [N]: VALID | FEASIBLE */
    /* chunk result */
    int64_t adm_idx, adm_delta, def_idx, def_delta;
    /* persistent worker: waits at `start`, scans, meets the driver at `done` */
    pthread_barrier_t *start, *done;
    volatile int32_t *quit;
} par_chunk;

static void *par_select_chunk(void *arg) {
    par_chunk *C = (par_chunk *)arg;
    const or_inst *I = C->I;
    const int64_t n = I->n, V = I->V, Rb = n * (n + V);
    evalctx X;
    evalctx_init(&X, I, C->len, C->r);
    C->adm_idx = C->def_idx = -1;
    C->adm_delta = C->def_delta = 0;
    /* (u, w) = (m, t) in the relocate block, (m1, m2) in the swap block, stepped
     * along with idx (no division per index) */
    int64_t u, w;
    if (C->lo < Rb) { u = C->lo / (n + V); w = C->lo % (n + V); }
    else { u = (C->lo - Rb) / (n > 0 ? n : 1); w = (C->lo - Rb) % (n > 0 ? n : 1); }
    for (int64_t idx = C->lo; idx < C->hi; idx++) {
        if (idx == Rb) { u = 0; w = 0; }
        else if (idx > C->lo) {
            if (++w == (idx < Rb ? n + V : n)) { w = 0; u++; }
        }
        move_t mv;
        int64_t delta = 0;
        int32_t feas = 0, valid;
        int32_t fresh = 1;
        if (C->memo && !C->first) {
            /* routes the move reads: those of m and t (relocate) or m1 and m2 (swap) */
            int32_t ra = X.veh[u], rb;
            if (idx < Rb) rb = w < n ? X.veh[w] : (int32_t)(w - n);
            else rb = X.veh[w];
            fresh = (ra >= 0 && C->changed[ra]) || (rb >= 0 && C->changed[rb]);
        }
        if (fresh) {
            valid = eval_one(&X, C->len, C->r, idx, C->prm->mask, 0, &mv, &delta, &feas);
            if (C->memo) {
                C->m_delta[idx] = (int32_t)delta;
                C->m_flags[idx] = (uint8_t)((valid ? OR_FLAG_VALID : 0) | (valid && feas ? OR_FLAG_FEASIBLE : 0));
            }
        } else {
            valid = (C->m_flags[idx] & OR_FLAG_VALID) != 0;
            feas = (C->m_flags[idx] & OR_FLAG_FEASIBLE) != 0;
            delta = C->m_delta[idx];
            if (!valid || !feas) continue;
            /* skip the tabu test of a move that cannot be selected whatever its class
             * (strict '<', ascending scan): no smaller than both running minima, or no
             * smaller than an admissible one (an admissible move anywhere beats every
             * by-default move, so this chunk's by-default minimum is then never used) */
            if (C->adm_idx >= 0 && delta >= C->adm_delta) continue;
            if (C->prm->mode == OR_MODE_TABU)
                build_move(I, C->len, C->r, X.veh, X.pos, idx, C->prm->mask, &mv, X.ra, X.rb);  /* its pairs */
        }
        if (!valid || !feas) continue;
        int32_t admissible;
        if (C->prm->mode == OR_MODE_TABU)
            admissible = !is_tabu(I, &mv, C->E, C->it) || X.cur + delta < C->best_obj;
        else
            admissible = delta < 0;
        if (admissible) {
            if (C->adm_idx < 0 || delta < C->adm_delta) { C->adm_idx = idx; C->adm_delta = delta; }
        } else {
            if (C->def_idx < 0 || delta < C->def_delta) { C->def_idx = idx; C->def_delta = delta; }
        }
    }
    evalctx_free(&X);
    return NULL;
}

static void *par_worker(void *arg) {
    par_chunk *C = (par_chunk *)arg;
    for (;;) {
        pthread_barrier_wait(C->start);
        if (*C->quit) break;
        par_select_chunk(C);
        pthread_barrier_wait(C->done);
    }
    return NULL;
}

int32_t or_search_par(const or_inst *I, const int32_t *len0, const int32_t *r0, const or_params *prm,
                      int32_t threads, int32_t memo, int32_t *best_len, int32_t *best_r, int32_t *final_len,
                      int32_t *final_r, or_result *res, int64_t *tr_idx, int32_t *tr_delta, int64_t *tr_cur,
                      int64_t *tr_best, int32_t *tr_cls, int32_t *E_out) {
    int32_t n = I->n, V = I->V;
    if (threads < 1) threads = 1;
    size_t rs = sizeof(int32_t) * (size_t)V * (size_t)(n > 0 ? n : 1);
    int64_t N = or_move_space_size(I);
    int32_t *len = (int32_t *)malloc(sizeof(int32_t) * (size_t)V);
    int32_t *r = (int32_t *)malloc(rs);
    int32_t *E = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1) * (size_t)V);
    uint8_t *changed = (uint8_t *)calloc((size_t)V, 1);
    int32_t *m_delta = memo ? (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1)) : NULL;
    uint8_t *m_flags = memo ? (uint8_t *)malloc((size_t)(N > 0 ? N : 1)) : NULL;
    par_chunk *C = (par_chunk *)calloc((size_t)threads, sizeof(par_chunk));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    pthread_barrier_t bstart, bdone;
    volatile int32_t quit = 0;
    if (threads > 1) {
        pthread_barrier_init(&bstart, NULL, (unsigned)threads + 1);
        pthread_barrier_init(&bdone, NULL, (unsigned)threads + 1);
        for (int32_t q = 0; q < threads; q++) {
            C[q].start = &bstart; C[q].done = &bdone; C[q].quit = &quit;
            pthread_create(&th[q], NULL, par_worker, &C[q]);
        }
    }
    memcpy(len, len0, sizeof(int32_t) * (size_t)V);
    memcpy(r, r0, rs);
    for (int64_t k = 0; k < (int64_t)n * V; k++) E[k] = -1;

    memset(res, 0, sizeof(*res));
    res->kicks_applied = or_kick(I, len, r, prm->seed, prm->kick);
    int64_t cur = or_objective(I, len, r);
    int64_t best = cur;
    res->start_obj = cur;
    res->best_iter = -1;
    memcpy(best_len, len, sizeof(int32_t) * (size_t)V);
    memcpy(best_r, r, rs);
    int32_t it;
    for (it = 0; it < prm->max_iters; it++) {
        for (int32_t q = 0; q < threads; q++) {
            par_chunk *c = &C[q];
            c->I = I; c->len = len; c->r = r; c->prm = prm;
            c->E = prm->mode == OR_MODE_TABU ? E : NULL;
            c->it = it; c->best_obj = best;
            c->lo = N * q / threads; c->hi = N * (q + 1) / threads;
            c->memo = memo; c->first = it == 0; c->changed = changed;
            c->m_delta = m_delta; c->m_flags = m_flags;
            if (threads == 1) par_select_chunk(c);
        }
        if (threads > 1) {
            pthread_barrier_wait(&bstart);   /* workers scan their chunks */
            pthread_barrier_wait(&bdone);
        }
        /* merge in chunk order with select_move's strict '<' */
        int64_t adm_idx = -1, adm_delta = 0, def_idx = -1, def_delta = 0;
        for (int32_t q = 0; q < threads; q++) {
            if (C[q].adm_idx >= 0 && (adm_idx < 0 || C[q].adm_delta < adm_delta)) { adm_idx = C[q].adm_idx; adm_delta = C[q].adm_delta; }
            if (C[q].def_idx >= 0 && (def_idx < 0 || C[q].def_delta < def_delta)) { def_idx = C[q].def_idx; def_delta = C[q].def_delta; }
        }
        int32_t cls;
        int64_t delta, idx;
        if (adm_idx >= 0) { cls = 0; delta = adm_delta; idx = adm_idx; }
        else if (def_idx >= 0) { cls = 1; delta = def_delta; idx = def_idx; }
        else { cls = -1; delta = 0; idx = -1; }
        if (cls < 0) { res->stop_reason = 2; break; }
        if (cls == 1 && prm->mode == OR_MODE_NS) { res->stop_reason = 1; break; }
        if (cls == 1 && prm->strict_tabu_stop) { res->stop_reason = 2; break; }
        evalctx X;
        evalctx_init(&X, I, len, r);
        move_t mv;
        int64_t d2;
        int32_t f2;
        eval_one(&X, len, r, idx, prm->mask, 0, &mv, &d2, &f2);
        write_back(I, len, r, &mv, X.ra, X.rb);
        evalctx_free(&X);
        memset(changed, 0, (size_t)V);
        changed[mv.a] = 1;
        changed[mv.b] = 1;
        cur += delta;
        if (prm->mode == OR_MODE_TABU)
            for (int32_t k = 0; k < mv.n_pairs; k++)
                E[(int64_t)mv.from_m[k] * V + mv.from_v[k]] = it + prm->tenure;
        if (cur < best) {
            best = cur;
            res->best_iter = it;
            memcpy(best_len, len, sizeof(int32_t) * (size_t)V);
            memcpy(best_r, r, rs);
        }
        if (tr_idx) tr_idx[it] = idx;
        if (tr_delta) tr_delta[it] = (int32_t)delta;
        if (tr_cur) tr_cur[it] = cur;
        if (tr_best) tr_best[it] = best;
        if (tr_cls) tr_cls[it] = cls;
    }
    res->iters_done = it;
    res->best_obj = best;
    res->final_obj = cur;
    if (final_len) memcpy(final_len, len, sizeof(int32_t) * (size_t)V);
    if (final_r) memcpy(final_r, r, rs);
    if (E_out) memcpy(E_out, E, sizeof(int32_t) * (size_t)n * (size_t)V);
    if (threads > 1) {
        quit = 1;
        pthread_barrier_wait(&bstart);
        for (int32_t q = 0; q < threads; q++) pthread_join(th[q], NULL);
        pthread_barrier_destroy(&bstart);
        pthread_barrier_destroy(&bdone);
    }
    free(len); free(r); free(E); free(changed); free(m_delta); free(m_flags); free(C); free(th);
    return 0;
}
