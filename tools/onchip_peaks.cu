// onchip_peaks.cu -- on-chip ceilings of this B200 for the roofline of the move-evaluation
// kernels ("smem random-gather GB/s, INT32 op/s ... from microbenchmarks run
// on the box at the measured clock").  One persistent CTA of 1024 threads per SM; every rate is
// given per SM-cycle (from %clock64 inside the kernel: clock-independent) and per second (CUDA
// events around the launch).  Printed as one JSON object.
//
//   int_alu    : independent IADD3 chains only (ALU pipe)
//   int_mix    : IADD3 and IMAD (mad.lo with a run-time multiplier) in equal numbers (ALU + FMA pipes,
//                the mix the scorers are written for, score.cuh madd)
//   lds_seq    : conflict-free LDS.32 (lane i reads word i of a row): one 128-B wavefront per warp-load
//   lds_gather : uint16 gathers at pseudo-random addresses of a 64 KB table (the scorers' T / node-cost
//                reads): useful gathers per cycle and the wavefronts they cost
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/onchip_peaks tools/onchip_peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));          \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

constexpr int THREADS = 1024;

__device__ __forceinline__ uint32_t iadd3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("add.u32 %0, %1, %2;\n\tadd.u32 %0, %0, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// 8 independent chains per thread, `iters` rounds; mix = 0: 8 IADD3 per round, 1: 4 IADD3 + 4 IMAD
template <int MIX>
__global__ void __launch_bounds__(THREADS, 1) k_int(int iters, uint32_t one, uint32_t *sink, long long *cyc) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x * 7 + k;
    const uint32_t b = blockIdx.x, c = one;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (MIX && (k & 1)) a[k] = imad(a[k], one, c + k);
            else a[k] = iadd3(a[k], b, c);
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) x ^= a[k];
    if (x == 0x12345678u) sink[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// conflict-free LDS.32: 8 independent loads per round, lane-consecutive words of a 32 KB buffer
__global__ void __launch_bounds__(THREADS, 1) k_lds_seq(int iters, uint32_t *sink, long long *cyc) {
    __shared__ uint32_t buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0;
    uint32_t row = (warp * 8) % 248;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        uint32_t v[8];
        const uint32_t *p = buf + row * 32 + lane;   // rows row .. row+7 < 256: immediate offsets
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = p[k * 32];
#pragma unroll
        for (int k = 0; k < 8; k++) acc += v[k];
        row += 8 + (acc & 1);                        // data dependence keeps the loads inside the loop
        if (row >= 248) row -= 248;
    }
    __syncthreads();
    const long long t1 = clock64();
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// LDS.U16 with STRIDE halfwords between lanes (1: 32 lanes read 64 contiguous bytes; 2: one halfword of each of
// 32 consecutive words): is a sub-word shared load one wavefront, or two?
template <int STRIDE>
__global__ void __launch_bounds__(THREADS, 1) k_lds_u16(int iters, uint32_t *sink, long long *cyc) {
    __shared__ uint16_t buf[16384];
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) buf[i] = (uint16_t)(i * 40503u);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0;
    uint32_t row = (warp * 8) % 192;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        uint32_t v[8];
        const uint16_t *p = buf + row * 64 + lane * STRIDE;   // 64 halfwords per row
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = p[k * 64];
#pragma unroll
        for (int k = 0; k < 8; k++) acc += v[k];
        row += 8 + (acc & 1);
        if (row >= 192) row -= 192;
    }
    __syncthreads();
    const long long t1 = clock64();
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// uint16 gathers at pseudo-random offsets of a 64 KB table: 8 independent gathers per round
__global__ void __launch_bounds__(THREADS, 1) k_lds_gather(int iters, uint32_t *sink, long long *cyc) {
    extern __shared__ uint16_t tab[];   // 32768 entries
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) tab[i] = (uint16_t)(i * 40503u);
    __syncthreads();
    uint32_t s = threadIdx.x * 2654435761u + blockIdx.x * 97u + 1u;
    uint32_t acc = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = tab[((s >> (k * 2)) + k * 4099u) & 32767u];
#pragma unroll
        for (int k = 0; k < 8; k++) acc += v[k];
        s = s * 1664525u + 1013904223u + (acc & 1);
    }
    __syncthreads();
    const long long t1 = clock64();
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

struct Meas {
    double ms, cycles;
};

template <class F>
static int timed(F launch, int nsm, long long *dcyc, Meas *out) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    launch();   // warm-up
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<long long> c(nsm);
    CK(cudaMemcpy(c.data(), dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
    double avg = 0;
    for (long long x : c) avg += (double)x;
    out->ms = ms;
    out->cycles = avg / nsm;
    return 0;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int nsm = prop.multiProcessorCount;
    uint32_t *sink;
    long long *cyc;
    CK(cudaMalloc(&sink, THREADS * 4));
    CK(cudaMalloc(&cyc, nsm * sizeof(long long)));
    const double warps = (double)nsm * THREADS / 32;
    const int it_int = 200000, it_lds = 40000;
    Meas m_alu, m_mix, m_seq, m_gat, m_u1, m_u2;
    if (timed([&] { k_int<0><<<nsm, THREADS>>>(it_int, 1u, sink, cyc); }, nsm, cyc, &m_alu)) return 1;
    if (timed([&] { k_int<1><<<nsm, THREADS>>>(it_int, 1u, sink, cyc); }, nsm, cyc, &m_mix)) return 1;
    if (timed([&] { k_lds_seq<<<nsm, THREADS>>>(it_lds, sink, cyc); }, nsm, cyc, &m_seq)) return 1;
    if (timed([&] { k_lds_u16<1><<<nsm, THREADS>>>(it_lds, sink, cyc); }, nsm, cyc, &m_u1)) return 1;
    if (timed([&] { k_lds_u16<2><<<nsm, THREADS>>>(it_lds, sink, cyc); }, nsm, cyc, &m_u2)) return 1;
    CK(cudaFuncSetAttribute(k_lds_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    if (timed([&] { k_lds_gather<<<nsm, THREADS, 65536>>>(it_lds, sink, cyc); }, nsm, cyc, &m_gat)) return 1;
    // thread-level integer ops: IADD3 counts as one op (two adds in the PTX above fold into one IADD3;
    // verified in the SASS by tools/onchip_peaks.py); 8 ops per round
    const double ops_int = warps * 32 * 8.0 * it_int;
    const double loads = warps * 8.0 * it_lds;   // warp-level loads
    auto rate = [&](double units, const Meas &m) { return units / (m.ms / 1e3); };
    auto per_cyc = [&](double units, const Meas &m) { return units / nsm / m.cycles; };
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"threads_per_cta\": %d,\n", prop.name, nsm, THREADS);
    printf(" \"sm_clock_mhz_effective\": %.1f,\n", m_mix.cycles / (m_mix.ms * 1e3));
    printf(" \"int_alu\": {\"ops_per_s\": %.6g, \"lanes_per_sm_cycle\": %.3f, \"ms\": %.3f},\n",
           rate(ops_int, m_alu), per_cyc(ops_int, m_alu), m_alu.ms);
    printf(" \"int_mix\": {\"ops_per_s\": %.6g, \"lanes_per_sm_cycle\": %.3f, \"ms\": %.3f},\n",
           rate(ops_int, m_mix), per_cyc(ops_int, m_mix), m_mix.ms);
    printf(" \"lds_seq\": {\"bytes_per_s\": %.6g, \"bytes_per_sm_cycle\": %.3f, \"wavefronts_per_sm_cycle\": %.3f, \"ms\": %.3f},\n",
           rate(loads * 128, m_seq), per_cyc(loads * 128, m_seq), per_cyc(loads, m_seq), m_seq.ms);
    printf(" \"lds_u16_contiguous\": {\"warp_loads_per_sm_cycle\": %.4f, \"ms\": %.3f},\n", per_cyc(loads, m_u1), m_u1.ms);
    printf(" \"lds_u16_word_stride\": {\"warp_loads_per_sm_cycle\": %.4f, \"ms\": %.3f},\n", per_cyc(loads, m_u2), m_u2.ms);
    printf(" \"lds_gather_u16\": {\"gathers_per_s\": %.6g, \"gathers_per_sm_cycle\": %.3f, \"useful_bytes_per_s\": %.6g, "
           "\"warp_loads_per_sm_cycle\": %.4f, \"ms\": %.3f}}\n",
           rate(loads * 32, m_gat), per_cyc(loads * 32, m_gat), rate(loads * 64, m_gat), per_cyc(loads, m_gat),
           m_gat.ms);
    return 0;
}
