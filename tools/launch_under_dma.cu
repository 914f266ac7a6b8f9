// Device-side cost of queued stream commands (small kernels, memsets,
// stream-ordered malloc/free, graph replays), on an idle PCIe link and while
// another stream runs a 30 MB pinned host->device copy. Diagnostic for the
// prepare's target side, whose short kernels run while the source cloud is
// still being uploaded.
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/launch_under_dma.cu -o /tmp/lud && /tmp/lud
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));      \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

__global__ void k_spin(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}
__global__ void k_small(float* a, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] += 1.0f;
}

enum Mode { kKernel, kMemset, kAlloc, kGraph };

int main() {
    const int kN = 1 << 16, kCmds = 10, kReps = 30;
    const size_t kCopy = 30u << 20;
    float* a;
    void *host, *dev, *big;
    CK(cudaMalloc(&a, kN * sizeof(float)));
    CK(cudaMalloc(&dev, kCopy));
    CK(cudaMalloc(&big, 8u << 20));
    CK(cudaHostAlloc(&host, kCopy, 0));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, 0));
    unsigned long long thr = ~0ull;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    cudaStream_t sc, sk;
    CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
    cudaGraphExec_t gexec;
    {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(sk, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < kCmds; ++k) k_small<<<kN / 256, 256, 0, sk>>>(a, kN);
        CK(cudaStreamEndCapture(sk, &g));
        CK(cudaGraphInstantiate(&gexec, g, 0));
        CK(cudaGraphUpload(gexec, sk));
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const char* names[] = {"small kernel", "8 MB memset", "kernel + 2 malloc/free async", "kernel in a graph"};
    for (int mode = kKernel; mode <= kGraph; ++mode)
        for (int dma = 0; dma < 2; ++dma) {
            std::vector<float> us;
            for (int r = 0; r < kReps + 2; ++r) {
                CK(cudaDeviceSynchronize());
                if (dma) CK(cudaMemcpyAsync(dev, host, kCopy, cudaMemcpyHostToDevice, sc));
                k_spin<<<1, 1, 0, sk>>>(400000);  // ~200 us: what follows is queued before it runs
                CK(cudaEventRecord(e0, sk));
                if (mode == kGraph) {
                    CK(cudaGraphLaunch(gexec, sk));
                } else {
                    for (int k = 0; k < kCmds; ++k) {
                        if (mode == kMemset) {
                            CK(cudaMemsetAsync(big, 0xff, 8u << 20, sk));
                        } else if (mode == kAlloc) {
                            void *p, *q;
                            CK(cudaMallocAsync(&p, 1 << 20, sk));
                            CK(cudaMallocAsync(&q, 1 << 20, sk));
                            k_small<<<kN / 256, 256, 0, sk>>>(a, kN);
                            CK(cudaFreeAsync(p, sk));
                            CK(cudaFreeAsync(q, sk));
                        } else {
                            k_small<<<kN / 256, 256, 0, sk>>>(a, kN);
                        }
                    }
                }
                CK(cudaEventRecord(e1, sk));
                CK(cudaDeviceSynchronize());
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (r >= 2) us.push_back(ms * 1e3f / kCmds);
            }
            std::sort(us.begin(), us.end());
            std::printf("%-30s %-16s %6.2f us per command (median of %d)\n", names[mode],
                        dma ? "during H2D DMA" : "idle link", us[us.size() / 2], kReps);
        }
    return 0;
}
