// compact.cuh -- compact array-of-structs layout shared by the batched and the
// grid-wide kernels: views with the engine.cuh interface over the records
//   CS[x] (16 B): {w, pick | del << 16, svc_class0, svc_class1}   (constants)
//   RS[x] (16 B): {depc, inc, svco, endc | veh << 16}             (per replica)
//   LK[x] (4 B):  {succ | pred << 16}                             (per replica)
#pragma once
#include <cstdint>

#include "engine.cuh"

namespace airsched {

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline int padded_stride(int NL, int tbytes) {
    if (tbytes == 2) {            // row stride in halfwords = 2 * odd number of words
        int w = (NL + 1) / 2;
        if ((w & 1) == 0) w++;
        return 2 * w;
    }
    return (NL & 1) ? NL : NL + 1; // odd number of words
}

// Class-layer stride (halfwords) of the window scorers' node-cost table TD[c][x][t] (rows of
// padded_stride(S, 2)): an odd multiple of 16 words, so that the two class layers of one row x
// start 16 banks apart and 32 lanes reading consecutive slots t of either class hit 32 banks.
__host__ __device__ inline int td_layer(int S, int NL) {
    const int words = NL * padded_stride(S, 2) / 2;
    const int w = (words + 31) / 32 * 32 + 16;   // >= words, == 16 (mod 32)
    return 2 * (w - 32 >= words ? w - 32 : w);
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
    // no-wait variant (f3): NR[x] (16 B) = {arrival, suffix slack, position, position of the suffix minimum}
    Field<int32_t, 16, 0> arr;
    Field<int32_t, 16, 4> sl;
    Field<int32_t, 16, 8> pos;
    Field<int32_t, 16, 12> slp;
    int32_t *F;
    ET *E;
};

// Warp minimum of a 64-bit key with two 32-bit REDUX.MIN (sm_80+): the minimum high word, then
// the minimum low word among the lanes holding it -- two instructions instead of five 64-bit
// shuffle rounds (the key reductions sit on the per-iteration critical path of k_grid / k_batch).
__device__ __forceinline__ uint64_t wmin(uint64_t v) {
    const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
    const uint32_t mh = __reduce_min_sync(0xFFFFFFFFu, hi);
    const uint32_t ml = __reduce_min_sync(0xFFFFFFFFu, hi == mh ? lo : 0xFFFFFFFFu);
    return ((uint64_t)mh << 32) | ml;
}

template <class T>
__device__ __forceinline__ T bcast(T v) {
    return __shfl_sync(0xFFFFFFFFu, v, 0);
}

// FULL: every move kind enabled (move_mask == 15): the per-move mask test is compiled out.
// L (the shared-memory layout) and NLp are computed on the host and passed by value,
// so the offsets are kernel-parameter constants rather than live registers.
}  // namespace airsched
