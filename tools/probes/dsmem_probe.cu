// Probe: random 2-byte gathers from a 128 KiB shared table -- local
// ld.shared vs ld.shared::cluster (own CTA) vs a fraction of lookups sent to a
// partner CTA of a 4-CTA cluster (DSMEM).  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a dsmem_probe.cu -o dsmem_probe
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

constexpr int kThreads = 1024;
constexpr int kTable = 1 << 17;
constexpr int kSteps = 4096;

template <int MODE>   // 0 ld.shared, 1 ld.shared::cluster own, 2 remote fraction
__global__ void __launch_bounds__(1024, 1) probe(uint32_t remote_thr, unsigned long long* sink) {
    extern __shared__ __align__(128) unsigned char tab[];
    for (int i = threadIdx.x; i < kTable / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(tab)[i] = (i * 2654435761u) & 0x0FFE0FFEu;
    uint32_t my = 0, nrank = 1;
    if (MODE >= 1) {
        cg::cluster_group cl = cg::this_cluster();
        my = cl.block_rank();
        nrank = cl.num_blocks();
        cl.sync();
    } else {
        __syncthreads();
    }
    uint32_t base = uint32_t(__cvta_generic_to_shared(tab));
    uint32_t rbase[4];
    for (int r = 0; r < 4; ++r) {
        uint32_t a = base;
        if (MODE >= 1) asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(base), "r"(uint32_t(r % nrank)));
        rbase[r] = a;
    }
    uint32_t x = threadIdx.x * 747796405u + blockIdx.x * 2891336453u + 1u;
    uint32_t e = 0, acc = 0;
    for (int j = 0; j < kSteps; ++j) {
        x = x * 1664525u + 1013904223u;
        const uint32_t a = ((x >> 8) & 0x1F000u) | (e & 0xFFEu);
        uint16_t v;
        if (MODE == 0) {
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(base + a));
        } else {
            const uint32_t tgt = (MODE == 2 && (x & 0xFFFFu) < remote_thr) ? ((my + 1) & 3) : my;
            asm volatile("ld.shared::cluster.u16 %0, [%1];" : "=h"(v) : "r"(rbase[tgt & 3] + a));
        }
        e = v;
        acc += e;
    }
    if (MODE >= 1) cg::this_cluster().sync();
    if (acc == 0x12345) sink[0] = acc;
}

template <int MODE>
float run(uint32_t thr, int cluster, int grid = 148) {
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTable);
    if (cluster > 1) cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kTable;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, probe<MODE>, thr, sink);
    cudaEventRecord(a);
    for (int w = 0; w < 5; ++w) cudaLaunchKernelEx(&cfg, probe<MODE>, thr, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t err = cudaGetLastError();
    if (err) printf("error %s\n", cudaGetErrorString(err));
    cudaFree(sink);
    return ms / 5;
}

int main() {
    const double lookups = 148.0 * kThreads * kSteps;
    float t0 = run<0>(0, 1);
    printf("ld.shared                    %.3f ms  %.2f G lookups/s\n", t0, lookups / t0 / 1e6);
    for (int cl : {2, 4}) {
        const int grid = cl == 4 ? 132 : 148;
        const double lk = double(grid) * kThreads * kSteps;
        float t1 = run<1>(0, cl, grid);
        printf("ld.shared::cluster own (c%d)  %.3f ms  %.2f G lookups/s\n", cl, t1, lk / t1 / 1e6);
        for (double f : {0.01, 0.03, 0.05, 0.10}) {
            float t2 = run<2>(uint32_t(f * 65536), cl, grid);
            printf("remote %.0f%% (c%d)             %.3f ms  %.2f G lookups/s\n", f * 100, cl, t2, lk / t2 / 1e6);
        }
    }
    return 0;
}
