/*
 * oracle.h -- CPU ORACLE FOR arXiv 2002.11710 (air-EMS fleet scheduling).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load, call or link this.
 * It shares no code, header, table or constant with the CUDA library under
 * paper_2002_11710_b200/ (and include/airsched.h), and neither includes the
 * other.
 *
 * What it computes, written as
 * the plain definitions: a schedule is an explicit list of missions per
 * vehicle (the paper's Solution matrix, Alg. 1 line 5); every
 * move is evaluated by applying it to copies of the affected routes and
 * recomputing their cost (Eq. obj_s) and feasibility (con6-con9,
 * P:128-134, text P:97/P:148) from scratch.
 */
#ifndef AIRSCHED_ORACLE_H
#define AIRSCHED_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t NL;                    /* number of locations */
    int32_t NC;                    /* number of vehicle classes (matrix layers l) */
    const int32_t *T;              /* [NC][NL][NL] integer seconds */
    const uint8_t *class_is_heli;  /* [NC] */
    int32_t V;                     /* vehicles (routing units) */
    const int32_t *veh_loc;        /* [V] base location of vehicle v */
    const int32_t *veh_cls;        /* [V] class (matrix layer) of vehicle v: l = b_k */
    int32_t n;                     /* missions */
    const int32_t *pick;           /* [n] pickup location */
    const int32_t *del;            /* [n] delivery location */
    const int32_t *w;              /* [n] deadline w_n, seconds */
    const uint8_t *heli;           /* [n] rho = 1: helicopter required */
    int32_t P;                     /* flight limit p, seconds */
    int32_t DAY;                   /* return limit, seconds */
    int32_t no_wait;               /* f3 variant: depart on arrival instead of at w (reading #40) */
} or_inst;

/* A schedule: len[v] missions in route v, stored in r[v*n + 0 .. len[v]-1]. */

int64_t or_route_cost(const or_inst *I, int32_t v, const int32_t *route, int32_t L);
int32_t or_route_feasible(const or_inst *I, int32_t v, const int32_t *route, int32_t L);
int64_t or_objective(const or_inst *I, const int32_t *len, const int32_t *r);
/* 1 iff every mission appears exactly once and every route is feasible. */
int32_t or_schedule_feasible(const or_inst *I, const int32_t *len, const int32_t *r);

int64_t or_move_space_size(const or_inst *I);

/* Apply canonical move idx (O5) to a copy; returns 1 if the move is VALID under mask. */
int32_t or_apply_move(const or_inst *I, const int32_t *len, const int32_t *r, int64_t idx,
                      uint32_t mask, int32_t *len_out, int32_t *r_out);

enum { OR_FLAG_VALID = 1, OR_FLAG_FEASIBLE = 2, OR_FLAG_TABU = 4, OR_FLAG_ADMISSIBLE = 8,
       OR_FLAG_BYDEFAULT = 16 };
enum { OR_MODE_NS = 0, OR_MODE_TABU = 1 };

/* Evaluate every canonical index (O6-O9).  E may be NULL (no tabu state).
 * full != 0 recomputes the objective and feasibility of the whole schedule per
 * move instead of only the affected routes.  best_*: the selected move
 * (class 0 = admissible, 1 = by-default; -1 if nothing selectable). */
void or_eval_moves(const or_inst *I, const int32_t *len, const int32_t *r, int32_t mode,
                   const int32_t *E, int32_t it, int64_t best_obj, uint32_t mask, int32_t full,
                   int32_t *delta_out, uint8_t *flags_out,
                   int32_t *best_cls, int32_t *best_delta, int64_t *best_idx);

/* or_eval_moves' per-index delta/flags for idx[0..count) only. */
void or_eval_index_list(const or_inst *I, const int32_t *len, const int32_t *r, int32_t mode, const int32_t *E,
                        int32_t it, int64_t best_obj, uint32_t mask, int64_t count, const int64_t *idx,
                        int32_t *delta_out, uint8_t *flags_out);

typedef struct {
    int32_t mode, tenure, max_iters, kick, strict_tabu_stop, want_digest;
    uint32_t mask;
    uint64_t seed;
} or_params;

typedef struct {
    int64_t best_obj, final_obj, start_obj;
    int32_t best_iter, iters_done, stop_reason, kicks_applied;
} or_result;

/* NS (O11) / TS (O10) with the seeded kick (O12).  Schedules in/out as len/r.
 * trace arrays (nullable) hold max_iters entries each.  E_out (nullable) gets
 * the final tabu expiry matrix [n][V]. */
int32_t or_search(const or_inst *I, const int32_t *len0, const int32_t *r0, const or_params *prm,
                  int32_t *best_len, int32_t *best_r, int32_t *final_len, int32_t *final_r,
                  or_result *res, int64_t *tr_idx, int32_t *tr_delta, int64_t *tr_cur,
                  int64_t *tr_best, int32_t *tr_cls, uint64_t *tr_digest, int32_t *E_out);

/* The same search (NS / TS + kick) driven over `threads` contiguous index chunks,
 * optionally keeping unchanged moves' values between iterations (memo); no
 * digests.  Identical results to or_search (see oracle.c). */
int32_t or_search_par(const or_inst *I, const int32_t *len0, const int32_t *r0, const or_params *prm,
                      int32_t threads, int32_t memo, int32_t *best_len, int32_t *best_r, int32_t *final_len,
                      int32_t *final_r, or_result *res, int64_t *tr_idx, int32_t *tr_delta, int64_t *tr_cur,
                      int64_t *tr_best, int32_t *tr_cls, int32_t *E_out);

/* f1: the paper-literal (i, j) sweep of Alg. 2 / Alg. 3 (see oracle.c).  One
 * trace entry per (i, j) step, idx -1 when CurrentMin stayed empty. */
int32_t or_sweep(const or_inst *I, const int32_t *len0, const int32_t *r0, const or_params *prm,
                 int32_t *best_len, int32_t *best_r, or_result *res, int64_t *tr_idx, int32_t *tr_delta,
                 int64_t *tr_cur, int64_t *tr_best);

/* The kick alone (O12): returns the number of relocates applied. */
int32_t or_kick(const or_inst *I, int32_t *len, int32_t *r, uint64_t seed, int32_t kick);

/* Algorithm 1 (O13).  Returns 0 on success, 3 on INIT_FAILED. */
int32_t or_greedy(const or_inst *I, int32_t insert_mode, int32_t max_repairs,
                  int32_t *len_out, int32_t *r_out, int32_t *n_repairs, int32_t *order_out);

/* f2: Algorithm 1 with a seeded placement order (reading #41); seed 0 == or_greedy. */
int32_t or_greedy_seeded(const or_inst *I, int32_t insert_mode, int32_t max_repairs, uint64_t seed,
                         int32_t *len_out, int32_t *r_out, int32_t *n_repairs, int32_t *order_out);

uint64_t or_splitmix64_next(uint64_t *state);
uint64_t or_tabu_digest(const or_inst *I, const int32_t *E, int32_t it);

#ifdef __cplusplus
}
#endif
#endif
