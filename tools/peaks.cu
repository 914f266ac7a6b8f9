// tools/peaks.cu -- measured ceilings for the roofline of the registration
// path (SURVEY.md §8d "Peaks"): the scorer is a gather from
// an L2-resident working set, so its denominators are L2 sector throughput
// (random 32-B sectors and streaming), shared-memory bandwidth, FP32/FP64 FMA
// throughput, with the SM clock observed under each load (clock64 vs
// %globaltimer inside the kernel). One JSON object on stdout.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
//   tools/peaks > profiles/peaks.json
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));    \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct ClockRec {
    unsigned long long cycles, ns;
};

__device__ __forceinline__ void clock_begin(uint64_t& c0, uint64_t& t0) {
    c0 = clock64();
    t0 = gtimer();
}
__device__ __forceinline__ void clock_end(uint64_t c0, uint64_t t0, ClockRec* rec) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        rec->cycles = clock64() - c0;
        rec->ns = gtimer() - t0;
    }
}

// random 32-B sector gather: each lane loads 16 B (one sector) from a
// pseudo-random sector of an L2-resident buffer; U independent loads in flight
template <int U>
__global__ void k_l2_random(const float4* __restrict__ buf, uint32_t sectors_mask, int iters, float* sink,
                            ClockRec* rec) {
    uint64_t c0, t0;
    clock_begin(c0, t0);
    uint32_t x = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    float acc = 0.0f;
    for (int it = 0; it < iters; ++it) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x ^= x << 13;
            x ^= x >> 17;
            x ^= x << 5;
            v[u] = __ldcg(buf + 2 * (x & sectors_mask));  // 32-B sector = 2 float4
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
    }
    if (acc == 1234.5f) *sink = acc;
    clock_end(c0, t0, rec);
}

// streaming (coalesced) reads of an L2-resident buffer
__global__ void k_l2_stream(const float4* __restrict__ buf, int64_t n4, int iters, float* sink, ClockRec* rec) {
    uint64_t c0, t0;
    clock_begin(c0, t0);
    float acc = 0.0f;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int it = 0; it < iters; ++it)
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
            const float4 v = __ldcg(buf + i);
            acc += v.x + v.w;
        }
    if (acc == 1234.5f) *sink = acc;
    clock_end(c0, t0, rec);
}

// shared memory: conflict-free float4 reads, 8 independent per iteration
__global__ void k_smem(int iters, float* sink, ClockRec* rec) {
    __shared__ float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    uint64_t c0, t0;
    clock_begin(c0, t0);
    float acc = 0.0f;
    int base = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float4 v = s[(base + 256 * u) & 2047];
            acc += v.x + v.y + v.z + v.w;
        }
        base = (base + 32) & 2047;
    }
    if (acc == 1234.5f) *sink = acc;
    clock_end(c0, t0, rec);
}

template <typename T>
__global__ void k_fma(int iters, T* sink, ClockRec* rec) {
    uint64_t c0, t0;
    clock_begin(c0, t0);
    T a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = static_cast<T>(threadIdx.x + u);
    const T m = static_cast<T>(0.999999), c = static_cast<T>(1e-7);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = fma(a[u], m, c);
    }
    T s = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += a[u];
    if (s == static_cast<T>(1234.5)) *sink = s;
    clock_end(c0, t0, rec);
}

template <typename F>
double time_ms(F&& launch, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    launch();  // warm
    CK(cudaDeviceSynchronize());
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, static_cast<double>(ms));
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    float* sink = nullptr;
    ClockRec* rec = nullptr;
    CK(cudaMalloc(&sink, 64));
    CK(cudaMallocManaged(&rec, sizeof(ClockRec)));
    auto mhz = [&]() { return rec->ns ? 1e3 * static_cast<double>(rec->cycles) / static_cast<double>(rec->ns) : 0.0; };

    std::printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d", prop.name, sms, prop.l2CacheSize);
    // L2 random sector gather over several working-set sizes (all L2-resident);
    // the best of a sweep over loads in flight per lane and resident threads
    const int threads = 512, blocks = sms * 4;
    std::printf(", \"l2_random_sector\": [");
    const int64_t sizes_mb[] = {8, 32, 64};
    for (int k = 0; k < 3; ++k) {
        const int64_t bytes = sizes_mb[k] << 20;
        float4* buf = nullptr;
        CK(cudaMalloc(&buf, bytes));
        CK(cudaMemset(buf, 0, bytes));
        const uint32_t sectors = static_cast<uint32_t>(bytes / 32);  // power of two
        double best = 0.0, best_mhz = 0.0;
        int best_u = 0, best_b = 0;
        for (int bpsm : {2, 4}) {
            for (int u : {8, 16, 32}) {
                const int nb = sms * bpsm, iters = 512 / u;
                double ms = time_ms(
                    [&] {
                        if (u == 8) k_l2_random<8><<<nb, 2048 / bpsm>>>(buf, sectors - 1, iters, sink, rec);
                        if (u == 16) k_l2_random<16><<<nb, 2048 / bpsm>>>(buf, sectors - 1, iters, sink, rec);
                        if (u == 32) k_l2_random<32><<<nb, 2048 / bpsm>>>(buf, sectors - 1, iters, sink, rec);
                    },
                    5);
                const double loads = static_cast<double>(nb) * (2048 / bpsm) * iters * u;
                const double gbs = loads * 32.0 / (ms * 1e6);
                if (gbs > best) best = gbs, best_mhz = mhz(), best_u = u, best_b = bpsm;
            }
        }
        std::printf("%s{\"working_set_mb\": %lld, \"gbs\": %.1f, \"sectors_per_s\": %.4g, \"sm_mhz\": %.0f, "
                    "\"loads_in_flight_per_lane\": %d, \"ctas_per_sm\": %d}",
                    k ? ", " : "", static_cast<long long>(sizes_mb[k]), best, best / 32.0 * 1e9, best_mhz, best_u,
                    best_b);
        CK(cudaFree(buf));
    }
    std::printf("]");
    {
        const int64_t bytes = 32ll << 20;
        float4* buf = nullptr;
        CK(cudaMalloc(&buf, bytes));
        CK(cudaMemset(buf, 0, bytes));
        const int iters = 32;
        double ms = time_ms([&] { k_l2_stream<<<blocks, threads>>>(buf, bytes / 16, iters, sink, rec); }, 5);
        std::printf(", \"l2_stream\": {\"working_set_mb\": 32, \"gbs\": %.1f, \"sm_mhz\": %.0f}",
                    static_cast<double>(bytes) * iters / (ms * 1e6), mhz());
        CK(cudaFree(buf));
    }
    {
        const int iters = 4096;
        double ms = time_ms([&] { k_smem<<<sms * 4, 512>>>(iters, sink, rec); }, 5);
        const double bytes = static_cast<double>(sms) * 4 * 512 * iters * 8 * 16;
        std::printf(", \"smem\": {\"gbs\": %.1f, \"sm_mhz\": %.0f}", bytes / (ms * 1e6), mhz());
    }
    {
        const int iters = 1 << 14;
        double ms = time_ms([&] { k_fma<float><<<sms * 8, 256>>>(iters, sink, rec); }, 5);
        const double flop = 2.0 * sms * 8 * 256 * static_cast<double>(iters) * 8;
        std::printf(", \"fp32_fma\": {\"tflops\": %.2f, \"sm_mhz\": %.0f}", flop / (ms * 1e9), mhz());
    }
    {
        double* dsink = nullptr;
        CK(cudaMalloc(&dsink, 64));
        const int iters = 1 << 12;
        double ms = time_ms([&] { k_fma<double><<<sms * 8, 256>>>(iters, dsink, rec); }, 5);
        const double flop = 2.0 * sms * 8 * 256 * static_cast<double>(iters) * 8;
        std::printf(", \"fp64_fma\": {\"tflops\": %.2f, \"sm_mhz\": %.0f}", flop / (ms * 1e9), mhz());
        CK(cudaFree(dsink));
    }
    std::printf(", \"how\": \"tools/peaks.cu: best of 5 CUDA-event timings after a warm-up; L2 random = 16-B __ldcg "
                "loads of xorshift-random 32-B sectors counted as 32 B each, best over 8/16/32 loads in flight per lane "
                "and 2/4 CTAs of 1024/512 threads per SM; others at %d x %d threads; sm_mhz = clock64 / "
                "%%globaltimer of block 0 during the kernel\"}\n",
                blocks, threads);
    return 0;
}
