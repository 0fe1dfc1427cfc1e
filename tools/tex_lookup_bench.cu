// Probe (dev tool, not product code): do random 1-byte label lookups go
// faster through the texture path (tex1Dfetch on linear memory) than through
// ld.global?  Same loop shape as the gather: persistent 1024-thread CTAs, 16
// lookups in flight per lane, byte stores.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tex_lookup_bench tex_lookup_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__global__ void fill_targets(int32_t *t, int64_t n, uint32_t range)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t[i] = (int32_t)(mix((uint64_t)i) % range);
}
__global__ void fill_table(uint8_t *t, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t[i] = (uint8_t)(mix((uint64_t)i * 7 + 1) % 51);
}

template <int GU, int MODE>  // MODE 0: ld.global.nc.u8, 1: tex1Dfetch<uchar>, 2: tex1Dfetch<uchar4> (word, then byte select)
__global__ void __launch_bounds__(1024, 1)
k_lookup(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table, cudaTextureObject_t tex,
         uint8_t *__restrict__ cls)
{
    constexpr int STEP = 32 * GU;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t steps = arcs / STEP;
    for (int64_t st = gw; st < steps; st += warps) {
        const int32_t *tp = targets + st * STEP + lane;
        uint32_t t[GU];
#pragma unroll
        for (int i = 0; i < GU; i++)
            asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(t[i]) : "l"(tp + 32 * i));
        uint32_t c[GU];
#pragma unroll
        for (int i = 0; i < GU; i++) {
            if (MODE == 0) c[i] = __ldg(table + t[i]);
            if (MODE == 1) c[i] = tex1Dfetch<unsigned char>(tex, (int)t[i]);
            if (MODE == 2) {
                const uchar4 v = tex1Dfetch<uchar4>(tex, (int)(t[i] >> 2));
                const uint32_t w = v.x | (v.y << 8) | (v.z << 16) | (v.w << 24);
                c[i] = (w >> (8 * (t[i] & 3))) & 0xffu;
            }
        }
        uint8_t *cp = cls + st * STEP + lane;
#pragma unroll
        for (int i = 0; i < GU; i++) cp[32 * i] = (uint8_t)c[i];
    }
}

template <int MODE>
void run(const char *name, const int32_t *targets, int64_t arcs, const uint8_t *table, cudaTextureObject_t tex,
         uint8_t *cls, int sms)
{
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    k_lookup<16, MODE><<<sms, 1024>>>(targets, arcs, table, tex, cls);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int r = 0; r < 5; r++) k_lookup<16, MODE><<<sms, 1024>>>(targets, arcs, table, tex, cls);
    CK(cudaEventRecord(b));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= 5;
    printf("%-44s %8.3f ms  %8.1f G lookups/s\n", name, ms, arcs / ms * 1e-6);
}

int main()
{
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int64_t arcs = 1ll << 28;
    int32_t *targets;
    uint8_t *table, *cls;
    const int64_t tmax = 150ll << 20;
    CK(cudaMalloc(&targets, arcs * 4));
    CK(cudaMalloc(&table, tmax));
    CK(cudaMalloc(&cls, arcs));
    fill_table<<<1024, 256>>>(table, tmax);
    for (int64_t range : {1ll << 20, 16ll << 20, 150ll << 20}) {
        fill_targets<<<2048, 256>>>(targets, arcs, (uint32_t)range);
        CK(cudaDeviceSynchronize());
        cudaTextureObject_t tex1 = 0, tex4 = 0;
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = table;
        rd.res.linear.desc = cudaCreateChannelDesc<unsigned char>();
        rd.res.linear.sizeInBytes = (size_t)range;
        cudaTextureDesc td = {};
        td.readMode = cudaReadModeElementType;
        cudaError_t e1 = cudaCreateTextureObject(&tex1, &rd, &td, nullptr);
        rd.res.linear.desc = cudaCreateChannelDesc<uchar4>();
        cudaError_t e4 = cudaCreateTextureObject(&tex4, &rd, &td, nullptr);
        char name[128];
        snprintf(name, sizeof name, "ld.global.nc.u8 over %lld MB", (long long)(range >> 20));
        run<0>(name, targets, arcs, table, 0, cls, sms);
        if (e1 == cudaSuccess) {
            snprintf(name, sizeof name, "tex1Dfetch<uchar> over %lld MB", (long long)(range >> 20));
            run<1>(name, targets, arcs, table, tex1, cls, sms);
        } else printf("uchar texture over %lld MB: %s\n", (long long)(range >> 20), cudaGetErrorString(e1));
        if (e4 == cudaSuccess) {
            snprintf(name, sizeof name, "tex1Dfetch<uchar4> + select over %lld MB", (long long)(range >> 20));
            run<2>(name, targets, arcs, table, tex4, cls, sms);
        } else printf("uchar4 texture over %lld MB: %s\n", (long long)(range >> 20), cudaGetErrorString(e4));
        cudaGetLastError();
        if (tex1) cudaDestroyTextureObject(tex1);
        if (tex4) cudaDestroyTextureObject(tex4);
    }
    // per-SM or chip-wide limit?  The same ld.global lookups (16 MB table) from fewer CTAs.
    fill_targets<<<2048, 256>>>(targets, arcs, 16u << 20);
    CK(cudaDeviceSynchronize());
    for (int g : {37, 74, 111, 148}) {
        char name[128];
        snprintf(name, sizeof name, "ld.global.nc.u8 over 16 MB, %d CTAs", g);
        run<0>(name, targets, arcs, table, 0, cls, g);
    }
    printf("done\n");
    return 0;
}
