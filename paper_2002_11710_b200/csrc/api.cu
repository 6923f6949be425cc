// api.cu -- the C ABI (include/airsched.h): validation, host<->device
// marshalling, launch policy.  Every step of the search path runs in the
// kernels of kernels.cu; host code here only validates inputs, copies buffers
// and (for Alg. 1, as_init_greedy) makes the deadline-ordered placement
// decisions, delegating its repair iteration to the device evaluator.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include <nccl.h>
#include <nccl_device.h>

#include "airsched.h"
#include "engine.cuh"
#include "launch.h"

using namespace airsched;

static thread_local std::string g_err;

static as_status fail(as_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            return fail(_e == cudaErrorMemoryAllocation ? AS_ERR_OOM : AS_ERR_DEVICE, "%s: %s (%s:%d)", \
                        #expr, cudaGetErrorString(_e), __FILE__, __LINE__);                         \
    } while (0)

// ----------------------------------------------------------------- instance --
struct as_instance {
    uint64_t uid;
    int32_t NL, NC, V, n, n_bases, P, DAY;
    int32_t no_wait = 0;   // f3 variant (reading #40)
    std::vector<int32_t> T, base_loc, vbase, vcls, vloc, pick, del, w;
    std::vector<uint8_t> cls_heli, heli, vcls8;
    int32_t maxT = 0;
    int32_t tsym = 1;      // T[c][a][b] == T[c][b][a] for every layer
    int64_t tdmax = 0;     // max over c, x, m of T_c[x][pick_m] + T_c[pick_m][del_m]
};

static uint64_t g_uid = 1;

extern "C" as_status as_instance_create(const as_instance_desc *d, as_instance **out) {
    if (!d || !out) return fail(AS_ERR_INVALID_ARG, "null argument");
    const int64_t NL = d->n_locations, NC = d->n_classes, V = d->n_vehicles, n = d->n_missions, B = d->n_bases;
    if (NL < 1 || NC < 1 || NC > 4) return fail(AS_ERR_INVALID_ARG, "need n_locations >= 1 and 1 <= n_classes <= 4");
    if (V < 1 || B < 1 || n < 0) return fail(AS_ERR_INVALID_ARG, "need n_vehicles >= 1, n_bases >= 1, n_missions >= 0");
    if (n + V >= (1 << 20)) return fail(AS_ERR_INVALID_ARG, "n + V must be < 2^20");
    if (n * (n + V) + n * n >= 0xFFFFFFFFll) return fail(AS_ERR_INVALID_ARG, "move space must be < 2^32 - 1");
    if (NC * NL * NL > (int64_t)1 << 31) return fail(AS_ERR_INVALID_ARG, "travel matrix too large");
    if (!d->travel_s || !d->class_is_heli || !d->base_location || !d->vehicle_base || !d->vehicle_class)
        return fail(AS_ERR_INVALID_ARG, "null array");
    if (n > 0 && (!d->pickup_loc || !d->delivery_loc || !d->deadline_s || !d->heli_only))
        return fail(AS_ERR_INVALID_ARG, "null mission array");
    if (d->flight_limit_s <= 0 || d->day_length_s >= (1 << 30) || d->day_length_s < d->flight_limit_s)
        return fail(AS_ERR_INVALID_ARG, "need 0 < flight_limit_s <= day_length_s < 2^30 (SPEC S:117)");
    if (d->no_wait != 0 && d->no_wait != 1) return fail(AS_ERR_INVALID_ARG, "no_wait must be 0 or 1");
    std::unique_ptr<as_instance> I(new (std::nothrow) as_instance());
    if (!I) return fail(AS_ERR_OOM, "host allocation");
    I->NL = (int32_t)NL; I->NC = (int32_t)NC; I->V = (int32_t)V; I->n = (int32_t)n; I->n_bases = (int32_t)B;
    I->P = d->flight_limit_s; I->DAY = d->day_length_s; I->no_wait = d->no_wait;
    I->T.assign(d->travel_s, d->travel_s + NC * NL * NL);
    for (int64_t c = 0; c < NC; c++)
        for (int64_t a = 0; a < NL; a++)
            for (int64_t b = 0; b < NL; b++) {
                int32_t t = I->T[(c * NL + a) * NL + b];
                if (t < 0 || t >= (1 << 26)) return fail(AS_ERR_INVALID_ARG, "travel_s[%lld][%lld][%lld] = %d outside [0, 2^26)", (long long)c, (long long)a, (long long)b, t);
                if (a == b && t != 0) return fail(AS_ERR_INVALID_ARG, "travel_s diagonal must be 0 (S:35)");
                if (t > I->maxT) I->maxT = t;
            }
    for (int64_t c = 0; c < NC && I->tsym; c++)
        for (int64_t a = 0; a < NL && I->tsym; a++)
            for (int64_t b = a + 1; b < NL; b++)
                if (I->T[(c * NL + a) * NL + b] != I->T[(c * NL + b) * NL + a]) { I->tsym = 0; break; }
    I->cls_heli.assign(d->class_is_heli, d->class_is_heli + NC);
    I->base_loc.assign(d->base_location, d->base_location + B);
    for (auto x : I->base_loc)
        if (x < 0 || x >= NL) return fail(AS_ERR_INVALID_ARG, "base_location out of range");
    I->vbase.assign(d->vehicle_base, d->vehicle_base + V);
    I->vcls.assign(d->vehicle_class, d->vehicle_class + V);
    I->vloc.resize(V);
    for (int64_t v = 0; v < V; v++) {
        if (I->vbase[v] < 0 || I->vbase[v] >= B) return fail(AS_ERR_INVALID_ARG, "vehicle_base[%lld] out of range", (long long)v);
        if (I->vcls[v] < 0 || I->vcls[v] >= NC) return fail(AS_ERR_INVALID_ARG, "vehicle_class[%lld] out of range", (long long)v);
        I->vloc[v] = I->base_loc[I->vbase[v]];
    }
    I->vcls8.assign(I->vcls.begin(), I->vcls.end());
    if (n > 0) {
        I->pick.assign(d->pickup_loc, d->pickup_loc + n);
        I->del.assign(d->delivery_loc, d->delivery_loc + n);
        I->w.assign(d->deadline_s, d->deadline_s + n);
        I->heli.assign(d->heli_only, d->heli_only + n);
    }
    for (int64_t m = 0; m < n; m++) {
        if (I->pick[m] < 0 || I->pick[m] >= NL || I->del[m] < 0 || I->del[m] >= NL)
            return fail(AS_ERR_INVALID_ARG, "mission %lld location out of range", (long long)m);
        if (I->w[m] < 1 || I->w[m] > d->day_length_s)
            return fail(AS_ERR_INVALID_ARG, "deadline of mission %lld outside [1, day_length] (S:111)", (long long)m);
        if (I->heli[m] > 1) return fail(AS_ERR_INVALID_ARG, "heli_only must be 0/1");
    }
    // largest node cost d_c(x, m) = T_c[x][pick_m] + T_c[pick_m][del_m] (O2): the window scorers stage
    // these as uint16 (batch.cu), so they need tdmax <= 65535
    for (int64_t c = 0; c < NC; c++) {
        std::vector<int32_t> colmax(NL, 0);
        for (int64_t a = 0; a < NL; a++)
            for (int64_t b = 0; b < NL; b++) colmax[b] = std::max(colmax[b], I->T[(c * NL + a) * NL + b]);
        for (int64_t m = 0; m < n; m++)
            I->tdmax = std::max<int64_t>(I->tdmax, (int64_t)colmax[I->pick[m]] + I->T[(c * NL + I->pick[m]) * NL + I->del[m]]);
    }
    I->uid = __atomic_fetch_add(&g_uid, 1, __ATOMIC_RELAXED);
    *out = I.release();
    return AS_OK;
}

extern "C" void as_instance_destroy(as_instance *inst) { delete inst; }

extern "C" int64_t as_move_space_size(const as_instance *I) {
    if (!I) return -1;
    int64_t n = I->n, V = I->V;
    return n * (n + V) + n * n;
}

extern "C" int64_t as_valid_moves_per_iter(const as_instance *I) {
    if (!I) return -1;
    int64_t n = I->n, V = I->V;
    return n > 0 ? n * (n + V - 2) + n * (n - 1) / 2 : 0;
}

// Host view of a CSR schedule: per-vehicle mission lists.
struct HostSched {
    std::vector<std::vector<int32_t>> routes;
};

static as_status parse_csr(const as_instance *I, const int32_t *ptr, const int32_t *ms, bool allow_partial,
                           HostSched &S) {
    if (!ptr) return fail(AS_ERR_INVALID_ARG, "null route_ptr");
    if (ptr[0] != 0) return fail(AS_ERR_INVALID_ARG, "route_ptr[0] must be 0");
    int32_t total = ptr[I->V];
    if (total < 0 || total > I->n) return fail(AS_ERR_INVALID_ARG, "route_ptr[V] out of range");
    if (!allow_partial && total != I->n) return fail(AS_ERR_INVALID_ARG, "schedule must list every mission once");
    if (total > 0 && !ms) return fail(AS_ERR_INVALID_ARG, "null route_missions");
    std::vector<char> seen(I->n, 0);
    S.routes.assign(I->V, {});
    for (int v = 0; v < I->V; v++) {
        if (ptr[v + 1] < ptr[v]) return fail(AS_ERR_INVALID_ARG, "route_ptr must be non-decreasing");
        for (int i = ptr[v]; i < ptr[v + 1]; i++) {
            int32_t m = ms[i];
            if (m < 0 || m >= I->n) return fail(AS_ERR_INVALID_ARG, "mission id %d out of range", m);
            if (seen[m]) return fail(AS_ERR_INVALID_ARG, "mission %d listed twice (con1/con2)", m);
            seen[m] = 1;
            S.routes[v].push_back(m);
        }
    }
    return AS_OK;
}

// Host arithmetic for validation and Alg. 1 placement (not the search path).
static inline int64_t hT(const as_instance *I, int c, int a, int b) {
    return I->T[((int64_t)c * I->NL + a) * I->NL + b];
}
static inline int32_t h_end(const as_instance *I, int v, int x) { return x >= 0 ? I->del[x] : I->vloc[v]; }
static inline int64_t h_dm(const as_instance *I, int v, int x, int m) {   // d(x -> mission m), class of v
    int c = I->vcls[v];
    return hT(I, c, h_end(I, v, x), I->pick[m]) + hT(I, c, I->pick[m], I->del[m]);
}
static inline int64_t h_db(const as_instance *I, int v, int x) { return hT(I, I->vcls[v], h_end(I, v, x), I->vloc[v]); }

static void route_eval(const as_instance *I, int v, const std::vector<int32_t> &r, int64_t *cost, bool *feas) {
    if (r.empty()) { *cost = 0; *feas = true; return; }
    int64_t c = 0, dep = 0;
    bool ok = true;
    int prev = -1;
    for (int32_t m : r) {
        int64_t d = h_dm(I, v, prev, m);
        if (dep + d > I->w[m]) ok = false;
        if (I->heli[m] && !I->cls_heli[I->vcls[v]]) ok = false;
        c += d;
        dep = I->no_wait ? dep + d : I->w[m];   // depart at w_m, or on arrival (f3)
        prev = m;
    }
    int64_t d = h_db(I, v, prev);
    if (dep + d > I->DAY) ok = false;
    c += d;
    if (c > I->P) ok = false;
    *cost = c;
    *feas = ok;
}

extern "C" as_status as_schedule_check(const as_instance *I, const int32_t *ptr, const int32_t *ms, int32_t *feasible,
                                       int64_t *objective) {
    if (!I) return fail(AS_ERR_INVALID_ARG, "null instance");
    HostSched S;
    as_status st = parse_csr(I, ptr, ms, true, S);
    if (st != AS_OK) return st;
    int64_t total = 0;
    bool ok = ptr[I->V] == I->n;
    for (int v = 0; v < I->V; v++) {
        int64_t c;
        bool f;
        route_eval(I, v, S.routes[v], &c, &f);
        total += c;
        ok = ok && f;
    }
    if (feasible) *feasible = ok ? 1 : 0;
    if (objective) *objective = total;
    return AS_OK;
}

struct as_schedule {
    std::vector<int32_t> ptr, ms;
    int64_t objective = 0;
    int32_t feasible = 0;
};

extern "C" as_status as_schedule_from_routes(const as_instance *I, const int32_t *ptr, const int32_t *ms,
                                             int32_t allow_partial, as_schedule **out) {
    if (!I || !out) return fail(AS_ERR_INVALID_ARG, "null argument");
    if (allow_partial != 0 && allow_partial != 1) return fail(AS_ERR_INVALID_ARG, "allow_partial must be 0 or 1");
    HostSched S;
    as_status st = parse_csr(I, ptr, ms, allow_partial != 0, S);
    if (st != AS_OK) return st;
    as_schedule *s = new (std::nothrow) as_schedule;
    if (!s) return fail(AS_ERR_OOM, "host allocation");
    s->ptr.assign(ptr, ptr + I->V + 1);
    s->ms.assign(ms ? ms : ptr, ms ? ms + ptr[I->V] : ptr);
    as_schedule_check(I, ptr, ms, &s->feasible, &s->objective);
    *out = s;
    return AS_OK;
}

extern "C" as_status as_schedule_get(const as_schedule *s, int32_t *ptr, int32_t *ms, int64_t *objective,
                                     int32_t *feasible, int32_t *n_assigned) {
    if (!s) return fail(AS_ERR_INVALID_ARG, "null schedule");
    if (ptr) std::copy(s->ptr.begin(), s->ptr.end(), ptr);
    if (ms) std::copy(s->ms.begin(), s->ms.end(), ms);
    if (objective) *objective = s->objective;
    if (feasible) *feasible = s->feasible;
    if (n_assigned) *n_assigned = (int32_t)s->ms.size();
    return AS_OK;
}

extern "C" void as_schedule_destroy(as_schedule *s) { delete s; }

// ------------------------------------------------------------------ context --
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
};

struct InstDev {
    uint64_t uid = 0;
    DevInst d{};
    void *Tpad = nullptr;     // padded travel-time table (uint16 when every entry fits)
    int tpad_bytes = 4;
    std::vector<void *> allocs;
};

struct as_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int n_sm = 148;
    size_t max_smem = 0;
    std::map<const as_instance *, InstDev> insts;
    std::map<std::string, DevBuf> scratch;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evj = nullptr;
    cudaStream_t cap = nullptr;   // private non-blocking stream for graph capture (torch's may be legacy)
    bool timed = false;
    float last_ms = 0.f;
    int32_t batch_runs = -1, batch_n = 0, batch_V = 0;   // last as_batch_run
    int64_t launches = 0;
    size_t max_smem_hw = 0;                 // the device's opt-in limit (max_smem = min(this, AS_OPT_SMEM_LIMIT))
    int64_t opt[AS_OPT_COUNT];              // as_ctx_set_option overrides; OPT_UNSET = automatic
    unsigned long long xr_timeout_ns = 30000000000ull;   // fused sharded exchange: bound on a peer's wait
    void *phase_dev = nullptr;              // k_grid phase sums of the last timed launch (AS_OPT_PHASE_TIMES)
    int phase_ctas = 0;                     // its CTA count (per-CTA records, as_ctx_grid_cta_phases)
};

struct as_comm {
    int nranks = 1, rank = 0, device = 0;
    ncclComm_t nccl = nullptr;
    // symmetric window of the fused sharded kernel (set up on first use, collectively)
    int dev_state = 0;             // 0 untried, 1 ready, -1 unavailable (LSA team != all ranks)
    void *xbuf = nullptr;          // symmetric buffer (ncclMemAlloc) holding the [3][nranks] {key, tag} slots
    ncclWindow_t win = nullptr;
    unsigned epoch = 0;            // fused runs so far (identical on every rank: the calls are collective)
};

// Grid-kernel options of a fused sharded run (run_core).
struct GridXr {
    int nranks, rank;
    unsigned epoch;
    unsigned long long timeout_ns;
    ncclWindow_t win;
};

constexpr int64_t OPT_UNSET = INT64_MIN;

// An as_ctx_set_option override, or the automatic choice dflt.
static int opt_int(const as_ctx *ctx, int option, int dflt) {
    const int64_t v = ctx->opt[option];
    return v == OPT_UNSET ? dflt : (int)v;
}

#define NCCL_TRY(expr)                                                                              \
    do {                                                                                            \
        ncclResult_t _r = (expr);                                                                   \
        if (_r != ncclSuccess)                                                                      \
            return fail(AS_ERR_COMM, "%s: %s (%s:%d)", #expr, ncclGetErrorString(_r), __FILE__, __LINE__); \
    } while (0)

static as_status set_device(as_ctx *ctx) {
    CUDA_TRY(cudaSetDevice(ctx->device));
    return AS_OK;
}

extern "C" as_status as_ctx_create(int32_t device, void *stream, as_ctx **out) {
    if (!out) return fail(AS_ERR_INVALID_ARG, "null out");
    int count = 0;
    CUDA_TRY(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(AS_ERR_INVALID_ARG, "device %d not present (%d devices)", device, count);
    std::unique_ptr<as_ctx> c(new as_ctx());
    c->device = device;
    c->stream = (cudaStream_t)stream;
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) return fail(AS_ERR_DEVICE, "this build targets sm_100a (B200); device is sm_%d%d", prop.major, prop.minor);
    c->n_sm = prop.multiProcessorCount;
    c->max_smem = c->max_smem_hw = prop.sharedMemPerBlockOptin;
    for (int k = 0; k < AS_OPT_COUNT; k++) c->opt[k] = OPT_UNSET;
    CUDA_TRY(cudaEventCreate(&c->ev0));
    CUDA_TRY(cudaEventCreate(&c->ev1));
    CUDA_TRY(cudaEventCreateWithFlags(&c->evj, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
    *out = c.release();
    return AS_OK;
}

extern "C" as_status as_ctx_set_option(as_ctx *ctx, int32_t option, int64_t value) {
    if (!ctx) return fail(AS_ERR_INVALID_ARG, "null ctx");
    if (option < 0 || option >= AS_OPT_COUNT) return fail(AS_ERR_INVALID_ARG, "unknown option %d", option);
    if (value != OPT_UNSET && (value < -1 || value > (int64_t)1 << 40))
        return fail(AS_ERR_INVALID_ARG, "option %d: value %lld out of range", option, (long long)value);
    ctx->opt[option] = value;
    if (option == AS_OPT_SMEM_LIMIT)
        ctx->max_smem = value == OPT_UNSET ? ctx->max_smem_hw : std::min<size_t>(ctx->max_smem_hw, (size_t)std::max<int64_t>(0, value));
    if (option == AS_OPT_XR_TIMEOUT_MS)
        ctx->xr_timeout_ns = value == OPT_UNSET ? 30000000000ull : (unsigned long long)std::max<int64_t>(1, value) * 1000000ull;
    return AS_OK;
}

extern "C" as_status as_ctx_grid_phases(as_ctx *ctx, int64_t *out) {
    if (!ctx || !out) return fail(AS_ERR_INVALID_ARG, "null argument");
    if (!ctx->phase_dev) return fail(AS_ERR_INVALID_ARG, "no whole-GPU run with AS_OPT_PHASE_TIMES yet");
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(cudaMemcpy(out, ctx->phase_dev, 10 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    return AS_OK;
}

extern "C" as_status as_ctx_grid_cta_phases(as_ctx *ctx, int64_t *tile_ns, int32_t *smid, int32_t *n_ctas) {
    if (!ctx || !tile_ns || !smid || !n_ctas) return fail(AS_ERR_INVALID_ARG, "null argument");
    if (!ctx->phase_dev) return fail(AS_ERR_INVALID_ARG, "no whole-GPU run with AS_OPT_PHASE_TIMES yet");
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    int64_t buf[2 * 256];
    CUDA_TRY(cudaMemcpy(buf, (int64_t *)ctx->phase_dev + 16, sizeof(buf), cudaMemcpyDeviceToHost));
    const int nc = std::min(ctx->phase_ctas, 256);
    for (int c = 0; c < nc; c++) { tile_ns[c] = buf[c]; smid[c] = (int32_t)buf[256 + c]; }
    *n_ctas = nc;
    return AS_OK;
}

extern "C" as_status as_ctx_set_stream(as_ctx *ctx, void *stream) {
    if (!ctx) return fail(AS_ERR_INVALID_ARG, "null ctx");
    ctx->stream = (cudaStream_t)stream;
    return AS_OK;
}

extern "C" void as_ctx_destroy(as_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto &kv : ctx->insts)
        for (void *p : kv.second.allocs) cudaFree(p);
    for (auto &kv : ctx->scratch) cudaFree(kv.second.p);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->evj) cudaEventDestroy(ctx->evj);
    if (ctx->cap) cudaStreamDestroy(ctx->cap);
    delete ctx;
}

extern "C" float as_ctx_last_kernel_ms(const as_ctx *ctx) {
    if (!ctx || !ctx->timed) return -1.f;
    as_ctx *c = const_cast<as_ctx *>(ctx);
    if (cudaEventSynchronize(c->ev1) != cudaSuccess) return -1.f;
    float ms = -1.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    return ms;
}

extern "C" int64_t as_ctx_kernel_launches(const as_ctx *ctx) { return ctx ? ctx->launches : -1; }

static as_status scratch(as_ctx *ctx, const char *name, size_t bytes, void **out) {
    DevBuf &b = ctx->scratch[name];
    if (b.cap < bytes) {
        if (b.p) {
            cudaStreamSynchronize(ctx->stream);
            cudaFree(b.p);
            b.p = nullptr;
            b.cap = 0;
        }
        size_t cap = std::max<size_t>(bytes, 256);
        CUDA_TRY(cudaMalloc(&b.p, cap));
        b.cap = cap;
    }
    *out = b.p;
    return AS_OK;
}

template <class Tp>
static as_status dev_copy(InstDev &D, const std::vector<Tp> &v, const Tp **out, cudaStream_t st) {
    void *p = nullptr;
    size_t bytes = std::max<size_t>(v.size() * sizeof(Tp), 16);
    CUDA_TRY(cudaMalloc(&p, bytes));
    D.allocs.push_back(p);
    if (!v.empty()) CUDA_TRY(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(Tp), cudaMemcpyHostToDevice, st));
    *out = (const Tp *)p;
    return AS_OK;
}

static as_status get_dev_inst(as_ctx *ctx, const as_instance *I, const DevInst **out) {
    auto it = ctx->insts.find(I);
    if (it != ctx->insts.end() && it->second.uid == I->uid) {
        *out = &it->second.d;
        return AS_OK;
    }
    if (it != ctx->insts.end()) {
        for (void *p : it->second.allocs) cudaFree(p);
        ctx->insts.erase(it);
    }
    InstDev D;
    D.uid = I->uid;
    as_status st;
    cudaStream_t s = ctx->stream;
    if ((st = dev_copy(D, I->T, &D.d.T, s)) != AS_OK) return st;
    if ((st = dev_copy(D, I->vloc, &D.d.vloc, s)) != AS_OK) return st;
    if ((st = dev_copy(D, I->vcls, &D.d.vcls, s)) != AS_OK) return st;
    if ((st = dev_copy(D, I->vcls8, &D.d.vcls8, s)) != AS_OK) return st;
    if ((st = dev_copy(D, I->cls_heli, &D.d.cls_heli, s)) != AS_OK) return st;
    if ((st = dev_copy(D, I->pick, &D.d.pick, s)) != AS_OK) return st;
    if ((st = dev_copy(D, I->del, &D.d.del, s)) != AS_OK) return st;
    if ((st = dev_copy(D, I->w, &D.d.w, s)) != AS_OK) return st;
    if ((st = dev_copy(D, I->heli, &D.d.heli, s)) != AS_OK) return st;
    void *svc = nullptr;
    CUDA_TRY(cudaMalloc(&svc, std::max<size_t>((size_t)I->NC * I->n * 4, 16)));
    D.allocs.push_back(svc);
    CUDA_TRY(launch_svc(D.d.T, D.d.pick, D.d.del, (int32_t *)svc, I->n, I->NL, I->NC, s));
    ctx->launches += I->n > 0;
    D.d.svc = (const int32_t *)svc;
    D.d.n = I->n; D.d.V = I->V; D.d.NL = I->NL; D.d.NC = I->NC; D.d.P = I->P; D.d.DAY = I->DAY;
    D.d.maxT = I->maxT;
    D.d.no_wait = I->no_wait;
    D.d.svcpos = 1;
    for (int c = 0; c < I->NC; c++)
        for (int m = 0; m < I->n; m++)
            if (hT(I, c, I->pick[m], I->del[m]) <= 0) D.d.svcpos = 0;
    D.tpad_bytes = I->maxT <= 65535 ? 2 : 4;
    {
        const int NLp = padded_stride_host(I->NL, D.tpad_bytes);
        void *tp = nullptr;
        CUDA_TRY(cudaMalloc(&tp, (size_t)I->NC * I->NL * NLp * D.tpad_bytes + 16));
        D.allocs.push_back(tp);
        CUDA_TRY(launch_pad_table(D.d.T, tp, I->NC, I->NL, NLp, D.tpad_bytes, false, s));
        ctx->launches++;
        D.Tpad = tp;
        D.d.tsym = I->tsym;
        D.d.TpadT = tp;
        if (!I->tsym) {   // the scorers read T[c][x][y] for x varying as the transposed row (score.cuh)
            void *tt = nullptr;
            CUDA_TRY(cudaMalloc(&tt, (size_t)I->NC * I->NL * NLp * D.tpad_bytes + 16));
            D.allocs.push_back(tt);
            CUDA_TRY(launch_pad_table(D.d.T, tt, I->NC, I->NL, NLp, D.tpad_bytes, true, s));
            ctx->launches++;
            D.d.TpadT = tt;
        }
    }
    // node costs for the global-table scorers (score.cuh): only when the table is too large for
    // shared memory (it is then read from global memory) and every node cost fits 16 bits
    D.d.TDg = nullptr;
    {
        const int NLp = padded_stride_host(I->NL, D.tpad_bytes);
        const size_t tsm = (size_t)I->NC * I->NL * NLp * D.tpad_bytes;
        if (D.tpad_bytes == 2 && I->tdmax <= 65535 && tsm > ctx->max_smem_hw / 2 && I->n > 0 &&
            opt_int(ctx, AS_OPT_NODE_COSTS, 1) == 1) {
            void *td = nullptr;
            const size_t bytes = (size_t)I->NC * I->NL * (I->n + I->V) * 2 + 16;
            CUDA_TRY(cudaMalloc(&td, bytes));
            D.allocs.push_back(td);
            CUDA_TRY(launch_build_td(D.d.T, D.d.pick, D.d.del, D.d.vloc, (uint16_t *)td, I->n, I->V, I->NL, I->NC, s));
            ctx->launches++;
            D.d.TDg = (const uint16_t *)td;
        }
    }
    auto &slot = ctx->insts[I];
    slot = std::move(D);
    *out = &slot.d;
    return AS_OK;
}

extern "C" as_status as_instance_upload(as_ctx *ctx, const as_instance *I) {
    if (!ctx || !I) return fail(AS_ERR_INVALID_ARG, "null argument");
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    const DevInst *d;
    return get_dev_inst(ctx, I, &d);
}

// Pointer classification: device memory of any kind counts as "device".
static bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Input array -> device pointer (copies host arrays into named scratch).
static as_status dev_in(as_ctx *ctx, const char *name, const void *p, size_t bytes, const void **out) {
    if (!p || is_device_ptr(p)) {
        *out = p;
        return AS_OK;
    }
    void *d;
    as_status st = scratch(ctx, name, bytes, &d);
    if (st != AS_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *out = d;
    return AS_OK;
}

// Output array: device pointer to write into; *host_dst set when a D2H copy is needed.
struct OutBuf {
    void *dev = nullptr;
    void *host = nullptr;
    size_t bytes = 0;
};
static as_status dev_out(as_ctx *ctx, const char *name, void *p, size_t bytes, OutBuf &o) {
    o.bytes = bytes;
    if (!p) return AS_OK;
    if (is_device_ptr(p)) {
        o.dev = p;
        return AS_OK;
    }
    as_status st = scratch(ctx, name, bytes, &o.dev);
    if (st != AS_OK) return st;
    o.host = p;
    return AS_OK;
}
static as_status finish_out(as_ctx *ctx, std::initializer_list<OutBuf *> outs) {
    bool any = false;
    for (OutBuf *o : outs)
        if (o->host && o->bytes) {
            CUDA_TRY(cudaMemcpyAsync(o->host, o->dev, o->bytes, cudaMemcpyDeviceToHost, ctx->stream));
            any = true;
        }
    if (any) CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return AS_OK;
}

// ------------------------------------------------------------ eval (dump) ---
struct GState {
    RunViewG g;
};

static as_status alloc_gstate(as_ctx *ctx, const as_instance *I, bool with_E, RunViewG &G) {
    const size_t S = (size_t)I->n + I->V;
    void *p;
    size_t words = 14 * S + (size_t)I->V + (with_E ? (size_t)I->n * I->V : 0) + 16;
    as_status st = scratch(ctx, "gstate", words * 4, &p);
    if (st != AS_OK) return st;
    int32_t *b = (int32_t *)p;
    G.succ = b; b += S;
    G.pred = b; b += S;
    G.veh = b; b += S;
    G.endc = b; b += S;
    G.depc = b; b += S;
    G.inc = b; b += S;
    G.svco = b; b += S;
    G.pick_s = b; b += S;
    G.w_s = b; b += S;
    G.F = b; b += I->V;
    G.arr = b; b += S;
    G.sl = b; b += S;
    G.pos = b; b += S;
    G.slp = b; b += S;
    G.E = with_E ? b : nullptr;
    return AS_OK;
}

// Internal eval used by as_eval_moves and the greedy repair.
static as_status eval_core(as_ctx *ctx, const as_instance *I, const DevInst *D, const HostSched &S, int mode,
                           const int32_t *tabu_expiry, int it, int64_t cur, int64_t best, uint32_t mask,
                           int32_t *delta_out, uint8_t *flags_out, uint64_t *best_key) {
    std::vector<int32_t> ptr(I->V + 1, 0), ms;
    for (int v = 0; v < I->V; v++) {
        ms.insert(ms.end(), S.routes[v].begin(), S.routes[v].end());
        ptr[v + 1] = (int32_t)ms.size();
    }
    const void *dptr, *dms;
    as_status st;
    if ((st = dev_in(ctx, "eval_ptr", ptr.data(), ptr.size() * 4, &dptr)) != AS_OK) return st;
    if ((st = dev_in(ctx, "eval_ms", ms.empty() ? nullptr : ms.data(), ms.size() * 4, &dms)) != AS_OK) return st;
    RunViewG G;
    bool tabu = mode == AS_MODE_TABU && tabu_expiry;
    if ((st = alloc_gstate(ctx, I, tabu, G)) != AS_OK) return st;
    if (tabu) {
        const void *dE;
        size_t eb = (size_t)I->n * I->V * 4;
        if ((st = dev_in(ctx, "eval_E", tabu_expiry, eb, &dE)) != AS_OK) return st;
        if (dE != G.E) CUDA_TRY(cudaMemcpyAsync(G.E, dE, eb, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CUDA_TRY(launch_build_state(*D, (const int32_t *)dptr, (const int32_t *)dms, G, ctx->stream));
    ctx->launches++;
    const uint64_t N = (uint64_t)as_move_space_size(I);
    OutBuf od, of, ok;
    if ((st = dev_out(ctx, "eval_delta", delta_out, N * 4, od)) != AS_OK) return st;
    if ((st = dev_out(ctx, "eval_flags", flags_out, N, of)) != AS_OK) return st;
    void *dkey;
    if ((st = scratch(ctx, "eval_key", 8, &dkey)) != AS_OK) return st;
    CUDA_TRY(cudaMemsetAsync(dkey, 0xFF, 8, ctx->stream));
    if (!tabu) G.E = nullptr;
    CUDA_TRY(cudaEventRecord(ctx->ev0, ctx->stream));
    if (N > 0) {
        CUDA_TRY(launch_eval_dump(*D, G, mode == AS_MODE_TABU ? 1 : 0, it, cur, best, mask, (int32_t *)od.dev,
                                  (uint8_t *)of.dev, (unsigned long long *)dkey, N, ctx->n_sm, ctx->stream));
        ctx->launches++;
    }
    CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->timed = true;
    ok.dev = dkey;
    ok.host = best_key;
    ok.bytes = best_key ? 8 : 0;
    return finish_out(ctx, {&od, &of, &ok});
}

extern "C" as_status as_eval_moves(as_ctx *ctx, const as_instance *I, const int32_t *ptr, const int32_t *ms,
                                   int32_t mode, const int32_t *tabu_expiry, int32_t iter, int64_t best_obj,
                                   uint32_t move_mask, int32_t *delta_out, uint8_t *flags_out, uint64_t *best_key_out) {
    if (!ctx || !I) return fail(AS_ERR_INVALID_ARG, "null ctx/instance");
    if (mode != AS_MODE_NS && mode != AS_MODE_TABU) return fail(AS_ERR_INVALID_ARG, "mode must be NS or TABU");
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    HostSched S;
    if ((st = parse_csr(I, ptr, ms, true, S)) != AS_OK) return st;
    int64_t cur = 0;
    for (int v = 0; v < I->V; v++) {
        int64_t c;
        bool f;
        route_eval(I, v, S.routes[v], &c, &f);
        if (!f) return fail(AS_ERR_INFEASIBLE_START, "route %d of the schedule is infeasible", v);
        cur += c;
    }
    const DevInst *D;
    if ((st = get_dev_inst(ctx, I, &D)) != AS_OK) return st;
    return eval_core(ctx, I, D, S, mode, tabu_expiry, iter, cur, best_obj, move_mask, delta_out, flags_out,
                     best_key_out);
}

// --------------------------------------------------------------- search -----
static as_status pick_layout(as_ctx *ctx, const as_instance *I, bool tabu, int *T_smem, int *E_smem, size_t *smem) {
    const size_t lim = ctx->max_smem;
    const int n = I->n, V = I->V, NL = I->NL, NC = I->NC;
    struct Opt { bool t, e; } opts[4] = {{true, true}, {true, false}, {false, true}, {false, false}};
    for (auto o : opts) {
        bool e = o.e && tabu;
        size_t b = search_smem_bytes(n, V, NL, NC, o.t, e, I->no_wait != 0);
        if (b <= lim) {
            *T_smem = o.t;
            *E_smem = e;
            *smem = b;
            return AS_OK;
        }
    }
    return fail(AS_ERR_UNSUPPORTED, "instance too large for the per-CTA persistent kernel (n=%d, V=%d)", n, V);
}


// The window scorers' general-leg form blocks a row whose removal leaves route a over the
// flight limit by adding NEG (-2^29) to P - F_b (window.cuh win_reloc_record): exact only while
// P < 2^28 (validation allows up to 2^30 - 1), so larger limits take the FAST scorers.
#define WIN_P_OK (I->P < (1 << 28))

static as_status run_core(as_ctx *ctx, const as_instance *I, int32_t n_runs, const int32_t *start_ptr,
                          const int32_t *start_ms, int32_t shared_start, const as_run_params *P,
                          const uint64_t *seeds, as_run_result *results, int32_t *best_ptr, int32_t *best_ms,
                          as_trace_rec *trace, uint64_t *digest, int32_t *tabu_out, bool single,
                          const GridXr *xr = nullptr) {
    if (!P) return fail(AS_ERR_INVALID_ARG, "null params");
    if (P->mode != AS_MODE_NS && P->mode != AS_MODE_TABU) return fail(AS_ERR_INVALID_ARG, "mode must be NS or TABU");
    if (P->max_iters < 0 || P->tenure < 0 || P->kick < 0) return fail(AS_ERR_INVALID_ARG, "negative parameter");
    if (n_runs < 1) return fail(AS_ERR_INVALID_ARG, "n_runs must be >= 1");
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    const DevInst *D;
    if ((st = get_dev_inst(ctx, I, &D)) != AS_OK) return st;
    const bool tabu = P->mode == AS_MODE_TABU;
    const int n = I->n, V = I->V;
    int T_smem, E_smem;
    size_t smem;
    const bool kfit = pick_layout(ctx, I, tabu, &T_smem, &E_smem, &smem) == AS_OK;
    if (!kfit) { T_smem = 0; E_smem = 0; smem = 0; }
    const int force_T = opt_int(ctx, AS_OPT_T_SMEM, -1);
    if (force_T == 0 && T_smem) {
        T_smem = 0;
        smem = search_smem_bytes(n, V, I->NL, I->NC, false, E_smem, I->no_wait != 0);
    }
    SearchArgs A;
    memset(&A, 0, sizeof(A));
    A.inst = *D;
    A.one = 1;
    A.neg = -1;
    const size_t nst = shared_start ? 1 : (size_t)n_runs;
    const void *dp, *dm, *ds = nullptr;
    if ((st = dev_in(ctx, "start_ptr", start_ptr, nst * (V + 1) * 4, &dp)) != AS_OK) return st;
    if ((st = dev_in(ctx, "start_ms", start_ms, std::max<size_t>(nst * n * 4, 4), &dm)) != AS_OK) return st;
    if (seeds && (st = dev_in(ctx, "seeds", seeds, (size_t)n_runs * 8, &ds)) != AS_OK) return st;
    A.start_ptr = (const int32_t *)dp;
    A.start_ms = (const int32_t *)dm;
    A.shared_start = shared_start;
    A.seeds = (const uint64_t *)ds;
    A.seed = P->seed;
    A.kick = P->kick;
    A.tenure = P->tenure;
    A.max_iters = P->max_iters;
    A.strict_tabu_stop = P->strict_tabu_stop;
    A.mask = P->sweep ? 1u : P->move_mask;   // the sweep relocates between bases only
    A.sweep = P->sweep ? 1 : 0;
    A.T_smem = T_smem;
    A.E_smem = E_smem;
    if (tabu && !E_smem) {
        void *e;
        if ((st = scratch(ctx, "E_global", (size_t)n_runs * n * V * 4 + 4, &e)) != AS_OK) return st;
        A.E_global = (int32_t *)e;
    }
    OutBuf o_res, o_bp, o_bm, o_tr, o_dg, o_tb;
    as_run_result *res_dev_needed = results;
    if ((st = dev_out(ctx, "o_res", res_dev_needed, (size_t)n_runs * sizeof(as_run_result), o_res)) != AS_OK) return st;
    if ((st = dev_out(ctx, "o_bp", best_ptr, (size_t)n_runs * (V + 1) * 4, o_bp)) != AS_OK) return st;
    if ((st = dev_out(ctx, "o_bm", best_ms, std::max<size_t>((size_t)n_runs * n * 4, 4), o_bm)) != AS_OK) return st;
    const bool want_trace = trace && P->trace_level >= 1 && P->max_iters > 0;
    const bool want_digest = digest && tabu && P->trace_level >= 2 && P->max_iters > 0;
    if ((st = dev_out(ctx, "o_tr", want_trace ? trace : nullptr, (size_t)n_runs * P->max_iters * sizeof(as_trace_rec), o_tr)) != AS_OK) return st;
    if ((st = dev_out(ctx, "o_dg", want_digest ? digest : nullptr, (size_t)n_runs * P->max_iters * 8, o_dg)) != AS_OK) return st;
    if ((st = dev_out(ctx, "o_tb", tabu ? tabu_out : nullptr, std::max<size_t>((size_t)n_runs * n * V * 4, 4), o_tb)) != AS_OK) return st;
    if (best_ptr && !best_ms && n > 0) return fail(AS_ERR_INVALID_ARG, "best_ptr_out needs best_missions_out");
    A.results = (as_run_result *)o_res.dev;
    A.best_ptr = (int32_t *)o_bp.dev;
    A.best_ms = best_ptr ? (int32_t *)o_bm.dev : nullptr;
    A.trace = (as_trace_rec *)o_tr.dev;
    A.digest = (uint64_t *)o_dg.dev;
    A.tabu_out = (int32_t *)o_tb.dev;
    // single-result call: results struct is host memory and required
    A.n_runs = n_runs;
    // launch policy: single runs -> one CTA per run (k_search); batches -> one run
    // per warp with the instance shared per CTA (k_batch) when the compact layout fits.
    const int64_t N = as_move_space_size(I);
    const int S = n + V;
    const int tbytes = I->maxT <= 65535 ? 2 : 4;
    const int ebytes = (int64_t)P->max_iters + P->tenure < 32767 ? 2 : 4;
    // window scorers (window.cuh) for the batched kernel: every move kind, positive service legs, uint16 table,
    // V <= 32 (tabu bits), bounded tenure (tabu-write ring), not the sweep
    bool win = (P->move_mask & 15u) == 15u && tbytes == 2 && I->tdmax <= 65535 && V <= 32 && !P->sweep &&
               (!tabu || P->tenure <= WIN_MAX_TENURE) && opt_int(ctx, AS_OPT_WINDOW, 1) == 1 &&
               WIN_P_OK && !I->no_wait;
    size_t sh_b = 0, run_b = 0;
    // the no-wait variant's batched kernel keeps int32 expiries and per-slot arrival/slack records
    batch_smem(n, V, I->NL, I->NC, tbytes, I->no_wait ? 4 : ebytes, tabu, &sh_b, &run_b, win, P->tenure,
               I->tsym != 0, I->no_wait != 0);
    int rpc_fit = run_b > 0 && sh_b < ctx->max_smem ? (int)((ctx->max_smem - sh_b) / run_b) : 0;
    if (win) {   // the window path stages more per CTA (node-cost tables): keep it only if it still fits the runs
        const int need = (int)std::min<int64_t>(28, ((int64_t)n_runs + ctx->n_sm - 1) / ctx->n_sm);
        size_t sh0 = 0, rb0 = 0;
        batch_smem(n, V, I->NL, I->NC, tbytes, ebytes, tabu, &sh0, &rb0);
        const int fit0 = rb0 > 0 && sh0 < ctx->max_smem ? (int)((ctx->max_smem - sh0) / rb0) : 0;
        if (rpc_fit < need && fit0 > rpc_fit) {
            win = false;
            sh_b = sh0;
            run_b = rb0;
            rpc_fit = fit0;
        }
    }
    // the compact layout (k_batch, k_grid); the no-wait variant (f3) has the batched kernel (exact
    // per-move evaluation, one run per warp) and, for single runs, the per-CTA kernel k_search
    const bool compact_fits = I->NL <= 65535 && S <= 65535 && V <= 32767 && I->NC <= 2 && !digest;
    const bool compact_ok = compact_fits && !I->no_wait;
    if (P->sweep && I->no_wait) return fail(AS_ERR_UNSUPPORTED, "the sweep mode (f1) is not built for the no-wait variant");
    const int want_batch = opt_int(ctx, AS_OPT_BATCH_KERNEL, -1);
    // no-wait batches stay on k_search unless asked for (one run per warp measured slower there:
    // 4.3e10 vs 6.0e10 move evals/s at 4096 C3 runs, profiles/r02/README.md)
    bool use_batch = (compact_ok && rpc_fit >= 1 && (want_batch == 1 || (want_batch == -1 && !single) || P->sweep)) ||
                     (compact_fits && I->no_wait && rpc_fit >= 1 && want_batch == 1);
    if (P->sweep && !use_batch)
        return fail(AS_ERR_UNSUPPORTED, "the sweep mode runs on the batched kernel (compact layout required)");
    // single large instances: one persistent cooperative grid (k_grid)
    bool use_grid = false;
    GridArgs GA;
    memset(&GA, 0, sizeof(GA));
    size_t grid_smem = 0;
    int grid_blocks = 0;
    int grid_warps = GRID_WARPS;   // warps per CTA of the whole-GPU kernel (AS_OPT_GRID_WARPS)
    if (xr && !(single && compact_ok && !P->sweep))
        return fail(AS_ERR_UNSUPPORTED, "fused sharded run needs the compact layout");
    // the whole-GPU kernel also runs the no-wait variant (general scorers, engine.cuh's exact evaluation)
    if (single && (compact_ok || (compact_fits && I->no_wait && !xr)) && !P->sweep) {
        const int want_grid = xr ? 1 : opt_int(ctx, AS_OPT_GRID, -1);
        const bool kfits = kfit;
        // CTAs: one per single-row tile up to the SM count (an iteration's floor is one tile's
        // latency + the grid barrier + the apply; an SM scoring many tiles at once is issue-bound,
        // DESIGN.md §7); ONE CTA (no grid barrier) when one CTA's warps take every tile
        const int64_t tiles1 = (int64_t)((S + 127) / 128 + (n > 1 ? (n - 1 + 63) / 64 : 0)) * n + (n + 31) / 32;
        const int need_blocks = (int)std::min<int64_t>(ctx->n_sm, tiles1);   // tiles spread one per CTA first
        const bool big = N >= opt_int(ctx, AS_OPT_GRID_MIN, 100000) || tiles1 > GRID_WARPS;
        // small single runs: the same kernel on ONE CTA (no grid barrier)
        const bool one_cta = !big && kfits && want_grid != 1 && opt_int(ctx, AS_OPT_ONE_CTA, 1) == 1;
        if (want_grid == 1 || one_cta || (want_grid == -1 && (big || !kfits))) {
            auto &D = ctx->insts[I];
            const int tb = D.tpad_bytes;
            struct Opt { bool t, e; } gopts[4] = {{true, true}, {true, false}, {false, true}, {false, false}};
            const bool t_global = opt_int(ctx, AS_OPT_GRID_T_GLOBAL, 0) == 1;   // test options
            const bool e_global = opt_int(ctx, AS_OPT_GRID_E_GLOBAL, 0) == 1;
            // fits for any rows-per-tile G (the compact-list prefix sized for G = 1), else for G >= 16 (the G
            // chosen below is then at least 16); resized below for the chosen G
            int gfit = 1;
            for (int pass = 0; pass < 2 && !use_grid; pass++) {
                gfit = pass ? 16 : 1;
                for (auto o : gopts) {
                    if ((t_global && o.t) || (e_global && o.e)) continue;
                    size_t b = grid_smem_bytes(n, V, I->NL, I->NC, tb, tabu && tb == 2 ? ebytes : 4, o.t, o.e && tabu,
                                               tabu, false, gfit, I->no_wait != 0);
                    if (b <= ctx->max_smem) {
                        GA.T_smem = o.t;
                        GA.E_smem = o.e && tabu;
                        grid_smem = b;
                        use_grid = true;
                        break;
                    }
                }
            }
            if (use_grid) {
                GA.ebytes = ebytes;
                int coop = 0;
                cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
                use_grid = coop != 0;
                grid_blocks = one_cta ? 1 : std::max(1, std::min(std::min(ctx->n_sm, 256), opt_int(ctx, AS_OPT_GRID_BLOCKS,
                                                                                      want_grid == 1 ? ctx->n_sm : need_blocks)));
                if (xr) grid_blocks = std::max(1, std::min(std::min(ctx->n_sm, 256), opt_int(ctx, AS_OPT_GRID_BLOCKS, ctx->n_sm)));
                // small instances: ONE cluster of up to 16 CTAs (every CTA's key stored into every CTA's shared
                // memory + one cluster barrier, instead of a global atomic, the grid barrier and a global read)
                // when its warps take every tile within two rounds
                GA.cluster = 0;
                {
                    const int clo = opt_int(ctx, AS_OPT_GRID_CLUSTER, -1);
                    const bool ok = !xr && !one_cta && GA.T_smem && (GA.E_smem || !tabu) && !I->no_wait;
                    int cl = 0;
                    if (ok && clo >= 2) cl = (int)std::min<int64_t>(clo, 16);
                    else if (ok && clo == -1 && want_grid != 1 && tiles1 <= 2 * 16 * GRID_WARPS) cl = 16;
                    const bool full = (P->move_mask & 15u) == 15u && D.d.svcpos;
                    while (cl >= 2 &&
                           grid_cluster_capacity(tabu ? 1 : 0, tb, ebytes, full, cl, GRID_WARPS * 32, grid_smem) < 1)
                        cl /= 2;
                    if (cl >= 2) {
                        GA.cluster = cl;
                        grid_blocks = cl;
                    }
                }
                GA.Tglobal = D.Tpad;
                void *p;
                GA.phase_ns = nullptr;
                if (opt_int(ctx, AS_OPT_PHASE_TIMES, 0) == 1 && !I->no_wait) {   // (no phase timers for no-wait)
                    if ((st = scratch(ctx, "g_phase", (16 + 2 * 256) * 8, &p)) != AS_OK) return st;
                    CUDA_TRY(cudaMemsetAsync(p, 0, (16 + 2 * 256) * 8, ctx->stream));
                    ctx->phase_ctas = grid_blocks;
                    GA.phase_ns = (unsigned long long *)p;
                    ctx->phase_dev = p;
                }
                if ((st = scratch(ctx, "g_key", 3 * 8, &p)) != AS_OK) return st;
                GA.gkey = (unsigned long long *)p;
                CUDA_TRY(cudaMemsetAsync(p, 0xFF, 3 * 8, ctx->stream));
                if ((st = scratch(ctx, "g_bs", (size_t)S * 4, &p)) != AS_OK) return st;
                GA.BS = (int32_t *)p;
                if (tabu && !GA.E_smem) {
                    if ((st = scratch(ctx, "g_E", (size_t)n * V * 4 + 4, &p)) != AS_OK) return st;
                    GA.Eglobal = (int32_t *)p;
                    if ((st = scratch(ctx, "g_Et", (size_t)n * V * 4 + 4, &p)) != AS_OK) return st;
                    GA.Etglobal = (int32_t *)p;
                }
                // rows per tile: the tiles go round-robin over the warps, so an iteration costs about
                // ceil(tiles / warps) rounds of G rows; take the G that minimises that (plus a per-round
                // set-up of ~1.5 rows: measured G sweeps, profiles/r02/grid_g_sweep_*.jsonl), the larger G
                // on ties; at most 32 rows (one key block).
                // warps per CTA: 20, or 8 on one cluster (its 16 CTAs then hold a tile per warp, and the CTA barriers of
                // the apply wait for fewer warps: C2 +6 %, the C3 instance alone +5 %, kgrid_warps_cluster.jsonl)
                grid_warps = (int)std::max<int64_t>(1, std::min<int64_t>(GRID_WARPS, opt_int(ctx, AS_OPT_GRID_WARPS,
                                                                                     GA.cluster > 1 ? 8 : GRID_WARPS)));
                const int64_t warps_all = (int64_t)grid_blocks * grid_warps * (xr ? xr->nranks : 1);
                const int64_t nTC = (S + 127) / 128, nSC = n > 1 ? (n - 1 + 63) / 64 : 0, nAdj = (n + 31) / 32;
                const int gmax = GA.T_smem ? 256 : 32;
                double best_cost = 1e300;
                GA.compact = xr ? 0 : opt_int(ctx, AS_OPT_GRID_COMPACT, 1);   // one GPU: no empty swap tiles (score.cuh)
                GA.G = gfit;
                for (int g = gfit; g <= std::max(gmax, gfit) && g <= std::max(gfit, n); g++) {
                    const int64_t tiles = GA.compact ? (int64_t)grid_tile_count_compact(n, V, g)
                                                     : (nTC + nSC) * ((n + g - 1) / g) + nAdj;
                    const int64_t rounds = (tiles + warps_all - 1) / warps_all;
                    const double cost = (double)rounds * g + 1.5 * (double)rounds;   // per-tile set-up ~1.5 rows
                    if (cost <= best_cost) { best_cost = cost; GA.G = g; }
                }
                GA.G = std::max(gfit, opt_int(ctx, AS_OPT_GRID_G, GA.G));
                // shared memory for this G (the compact-list prefix and table shrink with it); the global-table
                // scorers add per-warp swap-row records when they fit
                {
                    const int eb = tabu && D.tpad_bytes == 2 ? ebytes : 4;
                    const bool nw = I->no_wait != 0;
                    grid_smem = grid_smem_bytes(n, V, I->NL, I->NC, D.tpad_bytes, eb, GA.T_smem, GA.E_smem, tabu, false,
                                                GA.G, nw);
                    const size_t bsr = grid_smem_bytes(n, V, I->NL, I->NC, D.tpad_bytes, eb, GA.T_smem, GA.E_smem, tabu,
                                                       true, GA.G, nw);
                    GA.swap_rec = !GA.T_smem && !nw && bsr <= ctx->max_smem && opt_int(ctx, AS_OPT_GRID_SWAP_REC, 1) == 1;
                    if (GA.swap_rec) grid_smem = bsr;
                }
                GA.tlo = 0;
                GA.thi = GA.compact ? grid_tile_count_compact(n, V, GA.G) : grid_tile_count(n, V, GA.G);
                if (xr) {   // this rank's slice of the tile list (same weighted plan as the sharded kernels)
                    shard_plan(n, V, GA.G, xr->nranks, xr->rank, &GA.tlo, &GA.thi, nullptr, nullptr);
                    GA.xr = 1;
                    GA.xr_nranks = xr->nranks;
                    GA.xr_rank = xr->rank;
                    GA.xr_epoch = xr->epoch;
                    GA.xr_timeout_ns = xr->timeout_ns;
                    GA.xr_win = xr->win;
                    if ((st = scratch(ctx, "g_key2", 3 * 8, &p)) != AS_OK) return st;
                    GA.gkey2 = (unsigned long long *)p;
                }
            }
        }
    }
    if (xr && !use_grid) return fail(AS_ERR_UNSUPPORTED, "fused sharded run: the state does not fit the grid kernel");
    if (opt_int(ctx, AS_OPT_VERBOSE, 0))
        fprintf(stderr, "[airsched] n=%d V=%d runs=%d single=%d -> %s (blocks %d, G %d, T_smem %d, E_smem %d, smem %zu)\n",
                n, V, n_runs, (int)single, use_grid ? (xr ? "k_grid fused-sharded" : GA.cluster > 1 ? "k_grid/cluster" : grid_blocks == 1 ? "k_grid/1CTA" : "k_grid") :
                use_batch ? (win ? "k_batch/window" : "k_batch") : "k_search", grid_blocks, GA.G, GA.T_smem, GA.E_smem,
                use_grid ? grid_smem : smem);
    CUDA_TRY(cudaEventRecord(ctx->ev0, ctx->stream));
    if (use_grid) {
        CUDA_TRY(launch_grid(A, GA, tabu ? 1 : 0, ctx->insts[I].tpad_bytes, grid_blocks, grid_warps * 32, grid_smem,
                             ctx->stream));
        ctx->launches += A.best_ptr ? 2 : 1;
        ctx->launches--;   // counted once below
    } else if (use_batch) {
        int rpc = (int)std::min<int64_t>(28, std::min<int64_t>(rpc_fit, (n_runs + ctx->n_sm - 1) / ctx->n_sm));
        rpc = std::max(1, opt_int(ctx, AS_OPT_RPC, rpc));
        rpc = std::min(rpc, std::min(28, rpc_fit));
        size_t smem_b = sh_b + (size_t)rpc * run_b;
        if (win && tabu) {   // the window path keeps each run's tabu matrix in global memory
            void *e;
            if ((st = scratch(ctx, "E_win", (size_t)n_runs * n * V * 4 + 4, &e)) != AS_OK) return st;
            A.E_global = (int32_t *)e;
        }
        CUDA_TRY(launch_batch(A, tabu ? 1 : 0, rpc, tbytes, ebytes, smem_b, ctx->stream, win));
    } else {
        if (!kfit) return fail(AS_ERR_UNSUPPORTED, "instance too large for the per-CTA kernel (n=%d, V=%d)", n, V);
        int threads;
        if (single) {
            int64_t t = 64;
            while (t < 1024 && t * 16 < N) t *= 2;
            threads = (int)t;
        } else {
            threads = 256;
        }
        threads = opt_int(ctx, AS_OPT_THREADS, threads);
        CUDA_TRY(launch_search(A, tabu ? 1 : 0, n_runs, threads, smem, ctx->stream));
    }
    ctx->launches++;
    CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->timed = true;
    return finish_out(ctx, {&o_res, &o_bp, &o_bm, &o_tr, &o_dg, &o_tb});
}

static as_status sharded_run(as_ctx *ctx, as_comm *comm, const as_instance *I, const int32_t *start_ptr,
                             const int32_t *start_ms, const as_run_params *P, as_run_result *result,
                             int32_t *best_ptr, int32_t *best_ms, as_trace_rec *trace, int32_t *tabu_out);

extern "C" as_status as_tabu_run(as_ctx *ctx, as_comm *comm, const as_instance *I, const int32_t *start_ptr,
                                 const int32_t *start_ms, const as_run_params *P, as_run_result *result,
                                 int32_t *best_ptr, int32_t *best_ms, as_trace_rec *trace, uint64_t *digest,
                                 int32_t *tabu_out) {
    if (!ctx || !I || !P || !result) return fail(AS_ERR_INVALID_ARG, "null argument");
    HostSched S;
    as_status st = parse_csr(I, start_ptr, start_ms, false, S);
    if (st != AS_OK) return st;
    int32_t feas;
    int64_t obj;
    as_schedule_check(I, start_ptr, start_ms, &feas, &obj);
    if (!feas) return fail(AS_ERR_INFEASIBLE_START, "start schedule is infeasible (SPEC S:348)");
    if ((comm || opt_int(ctx, AS_OPT_SHARDED, 0) == 1) && !P->sweep) {
        if (I->no_wait) return fail(AS_ERR_UNSUPPORTED, "the sharded path is not built for the no-wait variant");
        if (digest && P->trace_level >= 2) return fail(AS_ERR_UNSUPPORTED, "tabu digests are not produced by the sharded path");
        return sharded_run(ctx, comm, I, start_ptr, start_ms, P, result, best_ptr, best_ms, trace, tabu_out);
    }
    st = run_core(ctx, I, 1, start_ptr, start_ms, 0, P, nullptr, result, best_ptr, best_ms, trace, digest, tabu_out, true);
    if (st == AS_ERR_UNSUPPORTED && !P->sweep && !I->no_wait && !(digest && P->trace_level >= 2) && I->NL <= 65535 &&
        I->n + I->V <= 65535 && I->NC <= 2) {
        // no on-chip kernel holds this instance's state: the sharded kernels keep it in global
        // memory (L2-resident), here with one rank
        return sharded_run(ctx, nullptr, I, start_ptr, start_ms, P, result, best_ptr, best_ms, trace, tabu_out);
    }
    if (st != AS_OK) return st;
    if (result->stop_reason == AS_STOP_INFEASIBLE_START)
        return fail(AS_ERR_INFEASIBLE_START, "device rejected the start schedule");
    return AS_OK;
}

extern "C" as_status as_nbhd_run(as_ctx *ctx, as_comm *comm, const as_instance *I, const int32_t *start_ptr,
                                 const int32_t *start_ms, const as_run_params *P, as_run_result *result,
                                 int32_t *best_ptr, int32_t *best_ms, as_trace_rec *trace) {
    if (!P) return fail(AS_ERR_INVALID_ARG, "null params");
    as_run_params q = *P;
    q.mode = AS_MODE_NS;
    return as_tabu_run(ctx, comm, I, start_ptr, start_ms, &q, result, best_ptr, best_ms, trace, nullptr, nullptr);
}

extern "C" as_status as_batch_run(as_ctx *ctx, as_comm *comm, const as_instance *I, int32_t n_runs,
                                  const int32_t *start_ptr, const int32_t *start_ms, int32_t shared_start,
                                  const as_run_params *P, const uint64_t *seeds, as_run_result *results,
                                  int32_t *best_ptr, int32_t *best_ms, as_trace_rec *trace, int64_t *best_run_out) {
    if (!ctx || !I || !P) return fail(AS_ERR_INVALID_ARG, "null argument");
    if (!start_ptr) return fail(AS_ERR_INVALID_ARG, "null start");
    // the best-run key packs (best objective << 32 | global run): objective <= V * P and the
    // global run index must each fit 32 bits
    if ((int64_t)I->V * I->P >= (1ll << 31))
        return fail(AS_ERR_UNSUPPORTED, "V * flight_limit_s >= 2^31: the best-run key cannot hold the objective");
    if ((int64_t)(comm ? comm->nranks : 1) * n_runs >= (1ll << 32))
        return fail(AS_ERR_INVALID_ARG, "nranks * n_runs >= 2^32");
    // results are needed on the device for the best-run reduction
    as_run_result *res = results;
    if (!res || !is_device_ptr(res)) {
        void *p;
        as_status st = scratch(ctx, "batch_res", (size_t)n_runs * sizeof(as_run_result), &p);
        if (st != AS_OK) return st;
        res = (as_run_result *)p;
    }
    as_status st = run_core(ctx, I, n_runs, start_ptr, start_ms, shared_start, P, seeds, res, best_ptr, best_ms,
                            trace, nullptr, nullptr, false);
    if (st != AS_OK) return st;
    // best (objective, global run) over all ranks: on the device, NCCL MIN across ranks
    void *kp;
    if ((st = scratch(ctx, "batch_key", 8, &kp)) != AS_OK) return st;
    const int64_t offset = comm ? (int64_t)comm->rank * n_runs : 0;
    CUDA_TRY(launch_batch_best(res, n_runs, offset, (unsigned long long *)kp, ctx->stream));
    ctx->launches++;
    if (comm && comm->nranks > 1)
        NCCL_TRY(ncclAllReduce(kp, kp, 1, ncclUint64, ncclMin, comm->nccl, ctx->stream));
    ctx->batch_runs = n_runs;
    ctx->batch_n = I->n;
    ctx->batch_V = I->V;
    if (results && res != results) {
        CUDA_TRY(cudaMemcpyAsync(results, res, (size_t)n_runs * sizeof(as_run_result), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    }
    if (best_run_out) {
        unsigned long long k;
        CUDA_TRY(cudaMemcpyAsync(&k, kp, 8, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        *best_run_out = k == AS_KEY_NONE ? -1 : (int64_t)(k & 0xFFFFFFFFull);
    }
    return AS_OK;
}

extern "C" as_status as_batch_run_jobs(as_ctx *ctx, as_comm *comm, int32_t n_jobs, const as_job *jobs,
                                       const as_run_params *P, const uint64_t *seeds, as_run_result *results,
                                       int32_t *best_ptr, int32_t *best_ms, as_trace_rec *trace,
                                       int64_t *best_run_out) {
    if (!ctx || !jobs || !P || n_jobs < 1) return fail(AS_ERR_INVALID_ARG, "null argument or no jobs");
    if (P->mode != AS_MODE_NS && P->mode != AS_MODE_TABU) return fail(AS_ERR_INVALID_ARG, "mode must be NS or TABU");
    if (P->max_iters < 0 || P->tenure < 0 || P->kick < 0) return fail(AS_ERR_INVALID_ARG, "negative parameter");
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    const bool tabu = P->mode == AS_MODE_TABU;
    int64_t total = 0, bp_total = 0, bm_total = 0;
    int tbytes = 2;
    for (int j = 0; j < n_jobs; j++) {
        const as_instance *I = jobs[j].inst;
        if (!I || !jobs[j].start_ptr || jobs[j].n_runs < 1) return fail(AS_ERR_INVALID_ARG, "job %d: null instance/start or n_runs < 1", j);
        if (I->NL > 65535 || I->n + I->V > 65535 || I->V > 32767 || I->NC > 2 || I->no_wait)
            return fail(AS_ERR_UNSUPPORTED, "job %d: the multi-instance batch needs the compact layout (NL, n+V < 65536, <= 2 classes, waiting model)", j);
        if (I->maxT > 65535) tbytes = 4;
        if ((int64_t)I->V * I->P >= (1ll << 31))   // best-run key: objective << 32 (see as_batch_run)
            return fail(AS_ERR_UNSUPPORTED, "job %d: V * flight_limit_s >= 2^31", j);
        total += jobs[j].n_runs;
        bp_total += (int64_t)jobs[j].n_runs * (I->V + 1);
        bm_total += (int64_t)jobs[j].n_runs * I->n;
    }
    if (total >= (1ll << 31) || (int64_t)(comm ? comm->nranks : 1) * total >= (1ll << 32))
        return fail(AS_ERR_INVALID_ARG, "too many runs");
    const int ebytes = (int64_t)P->max_iters + P->tenure < 32767 ? 2 : 4;
    // per-job device instance, layout, runs per CTA, packed start
    std::vector<BatchJob> J(n_jobs);
    std::vector<int4> cta;
    size_t smem = 0;
    int threads = 32;
    std::vector<int32_t> packed;           // host starts, uploaded once
    std::vector<std::pair<int64_t, int64_t>> poff(n_jobs, {-1, -1});
    // window scorers (window.cuh) for the FAST launch when every FAST job qualifies (V <= 32)
    bool win = ((P->sweep ? 1u : P->move_mask) & 15u) == 15u && !P->sweep && tbytes == 2 &&
               (!tabu || P->tenure <= WIN_MAX_TENURE) && opt_int(ctx, AS_OPT_WINDOW, 1) == 1 &&
               true;
    for (int j = 0; j < n_jobs && win; j++) {
        const DevInst *D;
        if ((st = get_dev_inst(ctx, jobs[j].inst, &D)) != AS_OK) return st;
        if (jobs[j].inst->V > 32 || jobs[j].inst->tdmax > 65535 || jobs[j].inst->P >= (1 << 28)) win = false;
    }
    int64_t run0 = 0, bp0 = 0, bm0 = 0, e0 = 0;
    for (int j = 0; j < n_jobs; j++) {
        const as_instance *I = jobs[j].inst;
        const DevInst *D;
        if ((st = get_dev_inst(ctx, I, &D)) != AS_OK) return st;
        BatchJob &b = J[j];
        b.inst = *D;
        const bool wj = win;
        b.L = batch_layout_host(I->n, I->V, I->NL, I->NC, tbytes, ebytes, tabu, wj, P->tenure, I->tsym != 0);
        b.e_off = e0;
        if (wj && tabu) e0 += (int64_t)jobs[j].n_runs * I->n * I->V;
        b.NLp = padded_stride_host(I->NL, tbytes);
        if ((size_t)b.L.shared_bytes + b.L.run_bytes > ctx->max_smem)
            return fail(AS_ERR_UNSUPPORTED, "job %d: instance too large for the batched kernel", j);
        const int fit = (int)((ctx->max_smem - b.L.shared_bytes) / b.L.run_bytes);
        {   // runs per CTA: as few CTAs as fit (<= 28 runs each), the job's runs spread evenly over them
            const int rmax = std::max(1, std::min(28, fit));
            const int nct = (jobs[j].n_runs + rmax - 1) / rmax;
            b.RPC = (jobs[j].n_runs + nct - 1) / nct;
        }
        b.run0 = (int)run0;
        b.bp_off = bp0;
        b.bm_off = bm0;
        if (is_device_ptr(jobs[j].start_ptr)) {
            b.start_ptr = jobs[j].start_ptr;
            b.start_ms = jobs[j].start_missions;
        } else {
            HostSched S;
            if ((st = parse_csr(I, jobs[j].start_ptr, jobs[j].start_missions, false, S)) != AS_OK) return st;
            poff[j].first = (int64_t)packed.size();
            packed.insert(packed.end(), jobs[j].start_ptr, jobs[j].start_ptr + I->V + 1);
            poff[j].second = (int64_t)packed.size();
            if (I->n > 0) packed.insert(packed.end(), jobs[j].start_missions, jobs[j].start_missions + I->n);
        }
        for (int r = 0; r < jobs[j].n_runs; r += b.RPC)
            cta.push_back(make_int4(j, r, std::min(b.RPC, jobs[j].n_runs - r), D->svcpos ? 1 : 0));
        smem = std::max(smem, (size_t)b.L.shared_bytes + (size_t)b.RPC * b.L.run_bytes);
        threads = std::max(threads, b.RPC * 32);
        run0 += jobs[j].n_runs;
        bp0 += (int64_t)jobs[j].n_runs * (I->V + 1);
        bm0 += (int64_t)jobs[j].n_runs * I->n;
    }
    if (!packed.empty()) {
        const void *dp;
        if ((st = dev_in(ctx, "jobs_starts", packed.data(), packed.size() * 4, &dp)) != AS_OK) return st;
        for (int j = 0; j < n_jobs; j++)
            if (poff[j].first >= 0) {
                J[j].start_ptr = (const int32_t *)dp + poff[j].first;
                J[j].start_ms = (const int32_t *)dp + poff[j].second;
            }
    }
    // the FAST scorers need every pickup->delivery leg > 0 (svcpos): with every move kind enabled the
    // CTAs of such jobs go first in one launch, the others in a second launch on a side stream
    const bool all_moves = ((P->sweep ? 1u : P->move_mask) & 15u) == 15u;
    std::stable_sort(cta.begin(), cta.end(), [&](const int4 &x, const int4 &y) { return (all_moves && x.w) > (all_moves && y.w); });
    int n_fast = 0;
    for (const int4 &c : cta) n_fast += all_moves && c.w;
    const void *djobs, *dcta, *ds = nullptr;
    if ((st = dev_in(ctx, "jobs_table", J.data(), J.size() * sizeof(BatchJob), &djobs)) != AS_OK) return st;
    if ((st = dev_in(ctx, "jobs_cta", cta.data(), cta.size() * sizeof(int4), &dcta)) != AS_OK) return st;
    if (seeds && (st = dev_in(ctx, "jobs_seeds", seeds, (size_t)total * 8, &ds)) != AS_OK) return st;
    as_run_result *res = results;
    if (!res || !is_device_ptr(res)) {
        void *p;
        if ((st = scratch(ctx, "jobs_res", (size_t)total * sizeof(as_run_result), &p)) != AS_OK) return st;
        res = (as_run_result *)p;
    }
    OutBuf o_bp, o_bm, o_tr;
    if (best_ptr && !best_ms && bm_total > 0) return fail(AS_ERR_INVALID_ARG, "best_ptr_out needs best_missions_out");
    if ((st = dev_out(ctx, "jobs_bp", best_ptr, (size_t)bp_total * 4, o_bp)) != AS_OK) return st;
    if ((st = dev_out(ctx, "jobs_bm", best_ptr ? best_ms : nullptr, std::max<size_t>((size_t)bm_total * 4, 4), o_bm)) != AS_OK) return st;
    const bool want_trace = trace && P->trace_level >= 1 && P->max_iters > 0;
    if ((st = dev_out(ctx, "jobs_tr", want_trace ? trace : nullptr, (size_t)total * P->max_iters * sizeof(as_trace_rec), o_tr)) != AS_OK) return st;
    SearchArgs A;
    memset(&A, 0, sizeof(A));
    A.one = 1;
    A.neg = -1;
    A.n_runs = (int32_t)total;
    A.seeds = (const uint64_t *)ds;
    A.seed = P->seed;
    A.kick = P->kick;
    A.tenure = P->tenure;
    A.max_iters = P->max_iters;
    A.strict_tabu_stop = P->strict_tabu_stop;
    A.mask = P->sweep ? 1u : P->move_mask;
    A.sweep = P->sweep ? 1 : 0;
    A.results = res;
    A.best_ptr = (int32_t *)o_bp.dev;
    A.best_ms = best_ptr ? (int32_t *)o_bm.dev : nullptr;
    A.trace = (as_trace_rec *)o_tr.dev;
    if (e0 > 0) {   // tabu matrices of the window-path runs (global memory)
        void *e;
        if ((st = scratch(ctx, "E_win_jobs", (size_t)e0 * 4 + 4, &e)) != AS_OK) return st;
        A.E_global = (int32_t *)e;
    }
    CUDA_TRY(cudaEventRecord(ctx->ev0, ctx->stream));
    const int n_gen = (int)cta.size() - n_fast;
    if (n_gen > 0 && n_fast > 0) {   // fork the general-scorer CTAs onto the side stream
        CUDA_TRY(cudaEventRecord(ctx->evj, ctx->stream));
        CUDA_TRY(cudaStreamWaitEvent(ctx->cap, ctx->evj, 0));
        CUDA_TRY(launch_batch_jobs(A, (const BatchJob *)djobs, (const int4 *)dcta + n_fast, n_gen, threads, smem,
                                   tabu ? 1 : 0, tbytes, ebytes, false, ctx->cap, win));
        ctx->launches++;
    }
    if (n_fast > 0) {
        CUDA_TRY(launch_batch_jobs(A, (const BatchJob *)djobs, (const int4 *)dcta, n_fast, threads, smem,
                                   tabu ? 1 : 0, tbytes, ebytes, true, ctx->stream, win));
        ctx->launches++;
    } else {
        CUDA_TRY(launch_batch_jobs(A, (const BatchJob *)djobs, (const int4 *)dcta, n_gen, threads, smem,
                                   tabu ? 1 : 0, tbytes, ebytes, false, ctx->stream, win));
        ctx->launches++;
    }
    if (n_gen > 0 && n_fast > 0) {   // join
        CUDA_TRY(cudaEventRecord(ctx->evj, ctx->cap));
        CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->evj, 0));
    }
    CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->timed = true;
    void *kp;
    if ((st = scratch(ctx, "batch_key", 8, &kp)) != AS_OK) return st;
    const int64_t offset = comm ? (int64_t)comm->rank * total : 0;
    CUDA_TRY(launch_batch_best(res, (int)total, offset, (unsigned long long *)kp, ctx->stream));
    ctx->launches++;
    if (comm && comm->nranks > 1)
        NCCL_TRY(ncclAllReduce(kp, kp, 1, ncclUint64, ncclMin, comm->nccl, ctx->stream));
    ctx->batch_runs = -1;   // as_batch_gather_best is for single-instance batches
    if (results && res != results)
        CUDA_TRY(cudaMemcpyAsync(results, res, (size_t)total * sizeof(as_run_result), cudaMemcpyDeviceToHost, ctx->stream));
    if ((st = finish_out(ctx, {&o_bp, &o_bm, &o_tr})) != AS_OK) return st;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (best_run_out) {
        unsigned long long k;
        CUDA_TRY(cudaMemcpyAsync(&k, kp, 8, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        *best_run_out = k == AS_KEY_NONE ? -1 : (int64_t)(k & 0xFFFFFFFFull);
    }
    return AS_OK;
}

extern "C" as_status as_batch_gather_best(as_ctx *ctx, as_comm *comm, int32_t n_runs, const int32_t *run_best_ptr,
                                          const int32_t *run_best_ms, int64_t *best_run_out, int64_t *best_obj_out,
                                          int32_t *ptr_out, int32_t *ms_out) {
    if (!ctx) return fail(AS_ERR_INVALID_ARG, "null ctx");
    if (ctx->batch_runs != n_runs) return fail(AS_ERR_INVALID_ARG, "no as_batch_run of %d runs on this context", n_runs);
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    void *kp;
    if ((st = scratch(ctx, "batch_key", 8, &kp)) != AS_OK) return st;
    unsigned long long k;
    CUDA_TRY(cudaMemcpyAsync(&k, kp, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const int64_t run = k == AS_KEY_NONE ? -1 : (int64_t)(k & 0xFFFFFFFFull);
    if (best_run_out) *best_run_out = run;
    if (best_obj_out) *best_obj_out = k == AS_KEY_NONE ? -1 : (int64_t)(k >> 32);
    if (!ptr_out || run < 0) return AS_OK;
    // owner copies its run's CSR into a buffer, NCCL broadcast to every rank
    const int rank = comm ? comm->rank : 0;
    const int owner = (int)(run / n_runs);
    const int r = (int)(run % n_runs);
    if (!run_best_ptr || !run_best_ms) return fail(AS_ERR_INVALID_ARG, "run_best_ptr/ms required for the schedule");
    const int V = ctx->batch_V, n = ctx->batch_n;
    void *buf;
    if ((st = scratch(ctx, "gbest", (size_t)(V + 1 + n) * 4 + 4, &buf)) != AS_OK) return st;
    if (rank == owner) {
        CUDA_TRY(cudaMemcpyAsync(buf, run_best_ptr + (size_t)r * (V + 1), (size_t)(V + 1) * 4, cudaMemcpyDefault, ctx->stream));
        if (n > 0)
            CUDA_TRY(cudaMemcpyAsync((int32_t *)buf + V + 1, run_best_ms + (size_t)r * n, (size_t)n * 4, cudaMemcpyDefault,
                                     ctx->stream));
    }
    if (comm && comm->nranks > 1)
        NCCL_TRY(ncclBroadcast(buf, buf, (size_t)(V + 1 + n), ncclInt32, owner, comm->nccl, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ptr_out, buf, (size_t)(V + 1) * 4, cudaMemcpyDefault, ctx->stream));
    if (n > 0 && ms_out)
        CUDA_TRY(cudaMemcpyAsync(ms_out, (int32_t *)buf + V + 1, (size_t)n * 4, cudaMemcpyDefault, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return AS_OK;
}

// ------------------------------------------------------------ Algorithm 1 ---
// Device Algorithm 1 for n_starts starts (greedy.cu, one warp per start).
extern "C" as_status as_init_greedy_batch(as_ctx *ctx, const as_instance *I, int32_t n_starts, int32_t insert_mode,
                                          int32_t max_repairs, const uint64_t *seeds, int32_t *route_ptr_out,
                                          int32_t *route_missions_out, int32_t *status_out, int32_t *n_repairs_out) {
    if (!ctx || !I || !route_ptr_out) return fail(AS_ERR_INVALID_ARG, "null argument");
    if (n_starts < 1) return fail(AS_ERR_INVALID_ARG, "n_starts must be >= 1");
    if (insert_mode != 0 && insert_mode != 1) return fail(AS_ERR_INVALID_ARG, "insert_mode must be 0 (TAIL) or 1 (SORTED)");
    if (max_repairs < 0) return fail(AS_ERR_INVALID_ARG, "max_repairs must be >= 0");
    if (I->n > 0 && !route_missions_out) return fail(AS_ERR_INVALID_ARG, "null route_missions_out");
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    const DevInst *D;
    if ((st = get_dev_inst(ctx, I, &D)) != AS_OK) return st;
    const int n = I->n, V = I->V;
    const size_t R = (size_t)n_starts;
    const void *ds = nullptr;
    if (seeds && (st = dev_in(ctx, "g_seeds", seeds, R * 8, &ds)) != AS_OK) return st;
    OutBuf op, om, os, onr;
    if ((st = dev_out(ctx, "g_ptr", route_ptr_out, R * (V + 1) * 4, op)) != AS_OK) return st;
    if ((st = dev_out(ctx, "g_ms", route_missions_out, std::max<size_t>(R * n * 4, 4), om)) != AS_OK) return st;
    if ((st = dev_out(ctx, "g_status", status_out, R * 4, os)) != AS_OK) return st;
    if ((st = dev_out(ctx, "g_nrep", n_repairs_out, R * 4, onr)) != AS_OK) return st;
    void *ord;
    if ((st = scratch(ctx, "g_order", (size_t)n * 4 + 4, &ord)) != AS_OK) return st;
    // layout: T + up to 8 warps of state in shared memory, else state only, else global state
    const size_t sb = greedy_state_bytes(*D);
    const size_t lim = ctx->max_smem;
    int warps = 0;
    bool T_smem = false, state_smem = false;
    if (opt_int(ctx, AS_OPT_GREEDY_GLOBAL, 0) == 1) warps = -1;   // test option: state in global memory
    for (int w = 8; w >= 1 && !warps; w /= 2)
        if (greedy_smem_bytes(*D, w, true, true) <= lim) { warps = w; T_smem = state_smem = true; }
    for (int w = 8; w >= 1 && !warps; w /= 2)
        if (greedy_smem_bytes(*D, w, false, true) <= lim) { warps = w; state_smem = true; }
    void *sg = nullptr;
    if (warps <= 0) {
        warps = 4;
        T_smem = greedy_smem_bytes(*D, warps, true, false) <= lim;
        if ((st = scratch(ctx, "g_state", R * sb, &sg)) != AS_OK) return st;
    }
    warps = std::max(1, std::min<int>(warps, (int)std::min<size_t>(8, R)));
    CUDA_TRY(cudaEventRecord(ctx->ev0, ctx->stream));
    CUDA_TRY(launch_greedy(*D, n_starts, insert_mode, max_repairs, (const uint64_t *)ds, (int32_t *)ord,
                           (int32_t *)sg, warps, T_smem, state_smem, (int32_t *)op.dev, (int32_t *)om.dev,
                           (int32_t *)os.dev, (int32_t *)onr.dev, ctx->stream));
    CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->timed = true;
    ctx->launches += n > 0 ? 2 : 1;
    return finish_out(ctx, {&op, &om, &os, &onr});
}

// Algorithm 1 for one start in the paper's order: the batched device kernel with n_starts = 1, seed 0.
extern "C" as_status as_init_greedy(as_ctx *ctx, const as_instance *I, int32_t insert_mode, int32_t max_repairs,
                                    int32_t *route_ptr_out, int32_t *route_missions_out, int32_t *n_repairs_out) {
    if (!ctx || !I || !route_ptr_out) return fail(AS_ERR_INVALID_ARG, "null argument");
    int32_t status = AS_OK, nrep = 0;
    as_status st = as_init_greedy_batch(ctx, I, 1, insert_mode, max_repairs, nullptr, route_ptr_out,
                                        route_missions_out, &status, &nrep);
    if (st != AS_OK) return st;
    if (status != AS_OK)
        return fail(AS_ERR_INIT_FAILED, "Algorithm 1: a mission could not be placed, even after %d repair(s) (P:166, P:213)", nrep);
    if (n_repairs_out) *n_repairs_out = nrep;
    return AS_OK;
}

// --------------------------------------------------------------- multi-GPU ---
extern "C" as_status as_comm_unique_id(void *uid_out) {
    if (!uid_out) return fail(AS_ERR_INVALID_ARG, "null uid_out");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    memcpy(uid_out, &id, sizeof(id));
    return AS_OK;
}

extern "C" as_status as_comm_init(as_ctx *ctx, int32_t nranks, int32_t rank, const void *uid, as_comm **out) {
    if (!ctx || !uid || !out) return fail(AS_ERR_INVALID_ARG, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(AS_ERR_INVALID_ARG, "bad rank %d of %d", rank, nranks);
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    std::unique_ptr<as_comm> c(new as_comm());
    c->nranks = nranks;
    c->rank = rank;
    c->device = ctx->device;
    NCCL_TRY(ncclCommInitRank(&c->nccl, nranks, id, rank));
    *out = c.release();
    return AS_OK;
}

extern "C" void as_comm_destroy(as_comm *comm) {
    if (!comm) return;
    if (comm->nccl) {
        cudaSetDevice(comm->device);
        if (comm->dev_state == 1) ncclCommWindowDeregister(comm->nccl, comm->win);
        if (comm->xbuf) ncclMemFree(comm->xbuf);
        ncclCommDestroy(comm->nccl);
    }
    delete comm;
}

static int shard_G(const as_instance *I, int n_sm) {
    const int n = I->n, V = I->V, S = n + V;
    const int warps_all = n_sm * 24;
    const int64_t nTC = (S + 127) / 128, nSC = n > 1 ? (n - 1 + 63) / 64 : 0;
    const int64_t pairs = (int64_t)n * nTC + (int64_t)n * nSC / 2;
    return (int)std::max<int64_t>(1, pairs / (4 * (int64_t)warps_all));
}

extern "C" as_status as_shard_plan(const as_instance *I, int32_t nranks, int32_t rank, int32_t n_sm, int32_t *tile_lo,
                                   int32_t *tile_hi, int32_t *tile_total, int64_t *weight_rank, int64_t *weight_total) {
    if (!I || nranks < 1 || rank < 0 || rank >= nranks || n_sm < 1) return fail(AS_ERR_INVALID_ARG, "bad argument");
    const int G = shard_G(I, n_sm);
    int lo, hi;
    int64_t wt, wr;
    shard_plan(I->n, I->V, G, nranks, rank, &lo, &hi, &wt, &wr);
    int last_lo, total;
    shard_plan(I->n, I->V, G, 1, 0, &last_lo, &total, nullptr, nullptr);
    if (tile_lo) *tile_lo = lo;
    if (tile_hi) *tile_hi = hi;
    if (tile_total) *tile_total = total;
    if (weight_rank) *weight_rank = wr;
    if (weight_total) *weight_total = wt;
    return AS_OK;
}

// Sharded single-instance run: replica in global memory, K iterations per CUDA
// graph of [eval slice -> ncclAllReduce(MIN, 8 B) -> apply].
// NCCL device-API state of a communicator (collective: every rank calls it in the same order).
// A one-word all-reduce (MIN) over the communicator on the legacy stream: the ranks agree on a flag
// and, as a side effect, meet (every rank's earlier stream work is complete when it returns).
static as_status comm_agree(as_comm *comm, int *flag) {
    int *d = nullptr;
    CUDA_TRY(cudaMalloc(&d, sizeof(int)));
    cudaError_t e = cudaMemcpy(d, flag, sizeof(int), cudaMemcpyHostToDevice);
    ncclResult_t r = e == cudaSuccess ? ncclAllReduce(d, d, 1, ncclInt32, ncclMin, comm->nccl, 0) : ncclSuccess;
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e == cudaSuccess) e = cudaMemcpy(flag, d, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (r != ncclSuccess) return fail(AS_ERR_COMM, "comm agreement: %s", ncclGetErrorString(r));
    if (e != cudaSuccess) return fail(AS_ERR_DEVICE, "comm agreement: %s", cudaGetErrorString(e));
    return AS_OK;
}

// The symmetric window of the fused sharded kernel (collective: every rank calls it in the same
// order).  Every step that can fail on one rank alone is followed by an agreement, so no rank enters
// the collective registration (or a fused kernel) while another has given up: on any failure all
// ranks fall back to the NCCL-graph path together.
static as_status comm_device_setup(as_comm *comm) {
    if (comm->dev_state) return AS_OK;
    comm->dev_state = -1;
    if (ncclTeamLsa(comm->nccl).nRanks != comm->nranks) return AS_OK;   // not every peer load/store reachable
    const size_t bytes = std::max<size_t>(4096, (size_t)3 * comm->nranks * 16);
    int ok = ncclMemAlloc(&comm->xbuf, bytes) == ncclSuccess;
    if (ok) ok = cudaMemset(comm->xbuf, 0, bytes) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
    as_status st = comm_agree(comm, &ok);   // tags 0 everywhere (no epoch >= 1 matches them) or nobody goes on
    if (st != AS_OK) return st;
    if (!ok) {
        if (comm->xbuf) ncclMemFree(comm->xbuf);
        comm->xbuf = nullptr;
        return AS_OK;
    }
    NCCL_TRY(ncclCommWindowRegister(comm->nccl, comm->xbuf, bytes, &comm->win, NCCL_WIN_COLL_SYMMETRIC));
    // every rank's window is zeroed and registered before any rank's first fused kernel can store into it
    int one = 1;
    if ((st = comm_agree(comm, &one)) != AS_OK) return st;
    comm->dev_state = 1;
    return AS_OK;
}

static as_status sharded_run(as_ctx *ctx, as_comm *comm, const as_instance *I, const int32_t *start_ptr,
                             const int32_t *start_ms, const as_run_params *P, as_run_result *result,
                             int32_t *best_ptr, int32_t *best_ms, as_trace_rec *trace, int32_t *tabu_out) {
    as_status st = set_device(ctx);
    if (st != AS_OK) return st;
    // Fused path (default with a communicator; AS_OPT_SHARD_FUSED = 0 disables it): one persistent
    // k_grid per rank scores the rank's tile slice and exchanges the 8-byte winner with its peers
    // through NVLink stores into a symmetric window (tagged slots, bounded wait) inside the kernel,
    // instead of [eval kernel, ncclAllReduce, apply kernel] per iteration.  Needs every peer in the LSA
    // team and the state in shared memory; otherwise the NCCL path below runs.
    if (comm && opt_int(ctx, AS_OPT_SHARD_FUSED, 1) == 1 && (comm->nranks > 1 || opt_int(ctx, AS_OPT_SHARD_FUSED_1, 0) == 1)) {
        if ((st = comm_device_setup(comm)) != AS_OK) return st;
        if (comm->dev_state == 1) {
            GridXr xr{comm->nranks, comm->rank, ++comm->epoch, ctx->xr_timeout_ns, comm->win};
            st = run_core(ctx, I, 1, start_ptr, start_ms, 0, P, nullptr, result, best_ptr, best_ms, trace, nullptr,
                          tabu_out, true, &xr);
            if (st == AS_OK && result->stop_reason == AS_STOP_COMM_ABORT)
                return fail(AS_ERR_COMM, "fused sharded run: a peer's key did not arrive within %.1f s (rank %d of %d)",
                            ctx->xr_timeout_ns / 1e9, comm->rank, comm->nranks);
            if (st != AS_ERR_UNSUPPORTED) return st;
        }
    }
    const DevInst *D;
    if ((st = get_dev_inst(ctx, I, &D)) != AS_OK) return st;
    InstDev &ID = ctx->insts[I];
    const bool tabu = P->mode == AS_MODE_TABU;
    const int n = I->n, V = I->V, S = n + V, NC = I->NC;
    if (I->NL > 65535 || S > 65535 || V > 32767 || NC > 2)
        return fail(AS_ERR_UNSUPPORTED, "sharded path needs NL, n+V < 65536 and <= 2 classes");
    SearchArgs A;
    memset(&A, 0, sizeof(A));
    A.inst = *D;
    A.one = 1;
    A.neg = -1;
    A.n_runs = 1;
    const void *dp, *dm;
    if ((st = dev_in(ctx, "start_ptr", start_ptr, (size_t)(V + 1) * 4, &dp)) != AS_OK) return st;
    if ((st = dev_in(ctx, "start_ms", start_ms, std::max<size_t>((size_t)n * 4, 4), &dm)) != AS_OK) return st;
    A.start_ptr = (const int32_t *)dp;
    A.start_ms = (const int32_t *)dm;
    A.shared_start = 1;
    A.seed = P->seed;
    A.kick = P->kick;
    A.tenure = P->tenure;
    A.max_iters = P->max_iters;
    A.strict_tabu_stop = P->strict_tabu_stop;
    A.mask = P->move_mask;
    // replica buffers
    ShardBufs B;
    void *p;
    size_t words = 0;
    const size_t oCS = 0, oRS = oCS + (size_t)S * 4, oLK = oRS + (size_t)S * 4, oF = oLK + S, oE = oF + V,
                 oBS = oE + (tabu ? (size_t)n * V : 0), oVC = oBS + S, oMH = oVC + V, oCH = oMH + (n + 3) / 4,
                 oCtl = oCH + 4;
    words = oCtl + (sizeof(ShardCtl) + 7) / 4 + 8;
    if ((st = scratch(ctx, "shard_state", words * 4 + 64, &p)) != AS_OK) return st;
    int32_t *base = (int32_t *)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    B.CS4 = (int4 *)(base + oCS);
    B.RS4 = (int4 *)(base + oRS);
    B.LK = (uint32_t *)(base + oLK);
    B.F = base + oF;
    B.E = tabu ? base + oE : nullptr;
    B.BS = base + oBS;
    B.VC = (uint32_t *)(base + oVC);
    B.MH = (uint8_t *)(base + oMH);
    B.CH = (uint8_t *)(base + oCH);
    B.ctl = (ShardCtl *)(((uintptr_t)(base + oCtl) + 15) & ~(uintptr_t)15);
    OutBuf o_res, o_bp, o_bm, o_tr, o_tb;
    if ((st = dev_out(ctx, "o_res", result, sizeof(as_run_result), o_res)) != AS_OK) return st;
    if ((st = dev_out(ctx, "o_bp", best_ptr, (size_t)(V + 1) * 4, o_bp)) != AS_OK) return st;
    if ((st = dev_out(ctx, "o_bm", best_ms, std::max<size_t>((size_t)n * 4, 4), o_bm)) != AS_OK) return st;
    const bool want_trace = trace && P->trace_level >= 1 && P->max_iters > 0;
    if ((st = dev_out(ctx, "o_tr", want_trace ? trace : nullptr, (size_t)P->max_iters * sizeof(as_trace_rec), o_tr)) != AS_OK) return st;
    if ((st = dev_out(ctx, "o_tb", tabu ? tabu_out : nullptr, std::max<size_t>((size_t)n * V * 4, 4), o_tb)) != AS_OK) return st;
    A.results = (as_run_result *)o_res.dev;
    A.best_ptr = best_ptr ? (int32_t *)o_bp.dev : nullptr;
    A.best_ms = best_ptr ? (int32_t *)o_bm.dev : nullptr;
    A.trace = (as_trace_rec *)o_tr.dev;
    A.tabu_out = (int32_t *)o_tb.dev;
    const int tb = ID.tpad_bytes;
    CUDA_TRY(launch_shard_init(A, B, ID.Tpad, tb, ctx->stream));
    ctx->launches++;
    const int nranks = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
    const int G = shard_G(I, ctx->n_sm);
    int tlo, thi;
    shard_plan(n, V, G, nranks, rank, &tlo, &thi, nullptr, nullptr);
    // Test mode (no communicator): emulate R ranks on one GPU by scoring the R
    // slices one after another into the same key before the apply.
    const int emulate = comm ? 1 : std::max(1, opt_int(ctx, AS_OPT_SHARD_EMULATE, 1));
    std::vector<std::pair<int, int>> slices;
    if (emulate > 1) {
        for (int r = 0; r < emulate; r++) {
            int a, b;
            shard_plan(n, V, G, emulate, r, &a, &b, nullptr, nullptr);
            slices.push_back({a, b});
        }
    } else {
        slices.push_back({tlo, thi});
    }
    // the iteration graphs run on the context's private capture stream, ordered
    // after everything already queued on cs
    cudaStream_t cs = ctx->cap;
    CUDA_TRY(cudaEventRecord(ctx->evj, ctx->stream));
    CUDA_TRY(cudaStreamWaitEvent(cs, ctx->evj, 0));
    CUDA_TRY(cudaEventRecord(ctx->ev0, cs));
    if (P->max_iters > 0) {
        const int K = std::max(1, std::min(P->max_iters, opt_int(ctx, AS_OPT_SHARD_K, 64)));
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < K; k++) {
            cudaError_t e1 = cudaSuccess;
            for (auto &sl : slices) {
                e1 = launch_shard_eval(A, B, ID.Tpad, tb, tabu ? 1 : 0, G, sl.first, sl.second, ctx->n_sm, cs);
                if (e1 != cudaSuccess) break;
            }
            if (e1 != cudaSuccess) { cudaStreamEndCapture(cs, &graph); return fail(AS_ERR_DEVICE, "shard eval: %s", cudaGetErrorString(e1)); }
            if (comm) {
                ncclResult_t r = ncclAllReduce(&B.ctl->key, &B.ctl->key, 1, ncclUint64, ncclMin, comm->nccl, cs);
                if (r != ncclSuccess) { cudaStreamEndCapture(cs, &graph); return fail(AS_ERR_COMM, "ncclAllReduce: %s", ncclGetErrorString(r)); }
            }
            e1 = launch_shard_apply(A, B, ID.Tpad, tb, tabu ? 1 : 0, cs);
            if (e1 != cudaSuccess) { cudaStreamEndCapture(cs, &graph); return fail(AS_ERR_DEVICE, "shard apply: %s", cudaGetErrorString(e1)); }
        }
        CUDA_TRY(cudaStreamEndCapture(cs, &graph));
        CUDA_TRY(cudaGraphInstantiate(&exec, graph, 0));
        int *hstop = nullptr;
        CUDA_TRY(cudaMallocHost(&hstop, sizeof(int)));
        const int chunks = (P->max_iters + K - 1) / K;
        for (int c = 0; c < chunks; c++) {
            cudaError_t e = cudaGraphLaunch(exec, cs);
            if (e == cudaSuccess) e = cudaMemcpyAsync(hstop, &B.ctl->stop, sizeof(int), cudaMemcpyDeviceToHost, cs);
            if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
            if (e != cudaSuccess) {
                cudaFreeHost(hstop);
                cudaGraphExecDestroy(exec);
                cudaGraphDestroy(graph);
                return fail(AS_ERR_DEVICE, "sharded iteration graph: %s", cudaGetErrorString(e));
            }
            ctx->launches += (int64_t)(slices.size() + 1) * K;
            if (*hstop) break;   // identical on every rank: all ranks apply the same keys
        }
        cudaFreeHost(hstop);
        CUDA_TRY(cudaGraphExecDestroy(exec));
        CUDA_TRY(cudaGraphDestroy(graph));
    }
    CUDA_TRY(cudaEventRecord(ctx->ev1, cs));
    ctx->timed = true;
    CUDA_TRY(cudaEventRecord(ctx->evj, cs));
    CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->evj, 0));
    CUDA_TRY(launch_shard_finish(A, B, ctx->stream));
    ctx->launches++;
    return finish_out(ctx, {&o_res, &o_bp, &o_bm, &o_tr, &o_tb});
}

extern "C" const char *as_last_error(void) { return g_err.c_str(); }
extern "C" const char *as_version(void) { return "airsched-b200 0.1 (sm_100a)"; }
