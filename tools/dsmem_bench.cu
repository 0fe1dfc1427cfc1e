// Random 1-byte lookup throughput: local shared memory, distributed shared
// memory across a thread-block cluster (ld via map_shared_rank), and global
// (L2-resident table).  Dev tool: does a cluster-pooled label head beat the
// L1->L2 request rate that bounds k_gather_tiered?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_bench tools/dsmem_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int THREADS = 1024;
constexpr int HEAD = 96 * 1024;
constexpr int ITERS = 256;
constexpr int MLP = 16;

__device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

// CS = cluster size (1: local smem only).  Each lookup picks a random byte of
// the pooled CS * HEAD bytes.
template <int CS>
__global__ void __launch_bounds__(THREADS, 1) k_dsmem(uint32_t *out, uint32_t seed)
{
    extern __shared__ __align__(16) unsigned char sm[];
    for (int i = threadIdx.x; i < HEAD / 4; i += THREADS) reinterpret_cast<uint32_t *>(sm)[i] = hash32(i + blockIdx.x);
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const unsigned char *base[CS];
#pragma unroll
    for (int r = 0; r < CS; r++) base[r] = cl.map_shared_rank(sm, r);
    uint32_t acc = 0, x = hash32(seed ^ (blockIdx.x * THREADS + threadIdx.x));
    for (int it = 0; it < ITERS; it++) {
        uint32_t v[MLP];
#pragma unroll
        for (int j = 0; j < MLP; j++) {
            x = hash32(x + j);
            const uint32_t slot = x % (uint32_t)(CS * HEAD);
            const uint32_t r = slot / HEAD, o = slot % HEAD;
            const unsigned char *p = base[0];
#pragma unroll
            for (int q = 1; q < CS; q++) p = (r == (uint32_t)q) ? base[q] : p;
            v[j] = p[o];
        }
#pragma unroll
        for (int j = 0; j < MLP; j++) acc += v[j];
    }
    cl.sync();
    if (acc == 0xdeadbeef) out[0] = acc;
}

__global__ void __launch_bounds__(THREADS, 1) k_global(const unsigned char *tab, uint32_t n, uint32_t *out, uint32_t seed)
{
    uint32_t acc = 0, x = hash32(seed ^ (blockIdx.x * THREADS + threadIdx.x));
    for (int it = 0; it < ITERS; it++) {
        uint32_t v[MLP];
#pragma unroll
        for (int j = 0; j < MLP; j++) {
            x = hash32(x + j);
            v[j] = __ldg(tab + x % n);
        }
#pragma unroll
        for (int j = 0; j < MLP; j++) acc += v[j];
    }
    if (acc == 0xdeadbeef) out[0] = acc;
}

template <int CS>
float run_cluster(int ctas, uint32_t *out)
{
    auto kern = k_dsmem<CS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, HEAD);
    if (CS > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas / CS * CS);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = HEAD;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, kern, out, 1u);
    cudaEventRecord(a);
    for (int i = 0; i < 5; i++) cudaLaunchKernelEx(&cfg, kern, out, (uint32_t)i + 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("cluster %d: %s\n", CS, cudaGetErrorString(e));
    const double lookups = 5.0 * (ctas / CS * CS) * THREADS * ITERS * MLP;
    printf("cluster %2d (%d CTAs): %.1f G lookups/s  (%.2f per SM clock at 1.9 GHz)\n", CS, ctas / CS * CS,
           lookups / (ms * 1e-3) / 1e9, lookups / (ms * 1e-3) / (ctas / CS * CS) / 1.9e9);
    return ms;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *out;
    cudaMalloc(&out, 4);
    run_cluster<1>(sms, out);
    run_cluster<2>(sms, out);
    run_cluster<4>(sms, out);
    run_cluster<8>(sms, out);
    run_cluster<16>(sms, out);
    for (uint32_t mb : {1u, 16u, 64u}) {
        const uint32_t n = mb << 20;
        unsigned char *tab;
        cudaMalloc(&tab, n);
        cudaMemset(tab, 1, n);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k_global<<<sms, THREADS>>>(tab, n, out, 1);
        cudaEventRecord(a);
        for (int i = 0; i < 5; i++) k_global<<<sms, THREADS>>>(tab, n, out, i + 2);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double lookups = 5.0 * sms * THREADS * ITERS * MLP;
        printf("global %u MB table: %.1f G lookups/s  (%.2f per SM clock)\n", mb, lookups / (ms * 1e-3) / 1e9,
               lookups / (ms * 1e-3) / sms / 1.9e9);
        cudaFree(tab);
    }
    return 0;
}
