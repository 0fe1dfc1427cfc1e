// Probe (dev tool, not product code): how fast can a persistent CTA stream
// targets, look their labels up in a shared-memory copy of one slot tile, and
// write a class byte per arc?  This is the upper bound for a tile-major heavy
// region (all lookups on chip).  Also: random 1-byte lookups that hit L1
// (tables of 16-64 KB) against lookups that go to L2 (16 MB).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tile_gather_bench tile_gather_bench.cu
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

// V0: lane-strided 32-bit target loads, byte table in shared memory, byte stores.
template <int GU>
__global__ void __launch_bounds__(1024, 1)
k_tile_bytes(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table, uint32_t slots,
             uint8_t *__restrict__ cls)
{
    extern __shared__ __align__(16) uint8_t tile[];
    for (uint32_t i = threadIdx.x; i < slots / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(tile)[i] = reinterpret_cast<const uint4 *>(table)[i];
    __syncthreads();
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
        uint8_t *cp = cls + st * STEP + lane;
#pragma unroll
        for (int i = 0; i < GU; i++) cp[32 * i] = tile[t[i]];
    }
}

// V1: each lane owns 4 consecutive arcs: 128-bit target loads, 32-bit class stores.
template <int GU4>
__global__ void __launch_bounds__(1024, 1)
k_tile_vec(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table, uint32_t slots,
           uint8_t *__restrict__ cls)
{
    extern __shared__ __align__(16) uint8_t tile[];
    for (uint32_t i = threadIdx.x; i < slots / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(tile)[i] = reinterpret_cast<const uint4 *>(table)[i];
    __syncthreads();
    constexpr int STEP = 128 * GU4;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t steps = arcs / STEP;
    for (int64_t st = gw; st < steps; st += warps) {
        const uint4 *tp = reinterpret_cast<const uint4 *>(targets + st * STEP) + lane;
        uint4 t[GU4];
#pragma unroll
        for (int i = 0; i < GU4; i++)
            asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(t[i].x), "=r"(t[i].y), "=r"(t[i].z), "=r"(t[i].w) : "l"(tp + 32 * i));
        uint32_t *cp = reinterpret_cast<uint32_t *>(cls + st * STEP) + lane;
#pragma unroll
        for (int i = 0; i < GU4; i++) {
            const uint32_t v = (uint32_t)tile[t[i].x] | ((uint32_t)tile[t[i].y] << 8) | ((uint32_t)tile[t[i].z] << 16) |
                               ((uint32_t)tile[t[i].w] << 24);
            cp[32 * i] = v;
        }
    }
}

// V2: 6-bit packed tile (5 labels per word), vector loads/stores.
template <int GU4>
__global__ void __launch_bounds__(1024, 1)
k_tile_packed(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table, uint32_t slots,
              uint8_t *__restrict__ cls)
{
    extern __shared__ __align__(16) uint32_t tw[];
    const uint32_t words = slots / 5;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) {
        uint32_t v = 0;
#pragma unroll
        for (int q = 0; q < 5; q++) v |= (uint32_t)table[i * 5 + q] << (6 * q);
        tw[i] = v;
    }
    __syncthreads();
    constexpr int STEP = 128 * GU4;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t steps = arcs / STEP;
    auto look = [&](uint32_t ti) {
        const uint32_t wi = ti / 5;
        return (tw[wi] >> (6 * (ti - wi * 5))) & 63u;
    };
    for (int64_t st = gw; st < steps; st += warps) {
        const uint4 *tp = reinterpret_cast<const uint4 *>(targets + st * STEP) + lane;
        uint4 t[GU4];
#pragma unroll
        for (int i = 0; i < GU4; i++)
            asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(t[i].x), "=r"(t[i].y), "=r"(t[i].z), "=r"(t[i].w) : "l"(tp + 32 * i));
        uint32_t *cp = reinterpret_cast<uint32_t *>(cls + st * STEP) + lane;
#pragma unroll
        for (int i = 0; i < GU4; i++)
            cp[32 * i] = look(t[i].x) | (look(t[i].y) << 8) | (look(t[i].z) << 16) | (look(t[i].w) << 24);
    }
}

// Global-memory lookups (L1 or L2 by table size), same loop shape as V0.
template <int GU>
__global__ void __launch_bounds__(1024, 1)
k_global_lookup(const int32_t *__restrict__ targets, int64_t arcs, const uint8_t *__restrict__ table,
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
        uint32_t l[GU];
#pragma unroll
        for (int i = 0; i < GU; i++)
            asm volatile("ld.global.nc.L1::evict_last.u8 %0, [%1];" : "=r"(l[i]) : "l"(table + t[i]));
        uint8_t *cp = cls + st * STEP + lane;
#pragma unroll
        for (int i = 0; i < GU; i++) cp[32 * i] = (uint8_t)l[i];
    }
}

// Plain copy of the two streams (4 B in, 1 B out per arc): the streaming bound of this loop shape.
template <int GU4>
__global__ void __launch_bounds__(1024, 1)
k_stream_only(const int32_t *__restrict__ targets, int64_t arcs, uint8_t *__restrict__ cls)
{
    constexpr int STEP = 128 * GU4;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t steps = arcs / STEP;
    for (int64_t st = gw; st < steps; st += warps) {
        const uint4 *tp = reinterpret_cast<const uint4 *>(targets + st * STEP) + lane;
        uint4 t[GU4];
#pragma unroll
        for (int i = 0; i < GU4; i++)
            asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(t[i].x), "=r"(t[i].y), "=r"(t[i].z), "=r"(t[i].w) : "l"(tp + 32 * i));
        uint32_t *cp = reinterpret_cast<uint32_t *>(cls + st * STEP) + lane;
#pragma unroll
        for (int i = 0; i < GU4; i++)
            cp[32 * i] = (t[i].x & 63u) | ((t[i].y & 63u) << 8) | ((t[i].z & 63u) << 16) | ((t[i].w & 63u) << 24);
    }
}

template <class F>
static float time_ms(F f, int reps = 5)
{
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    f();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; i++) f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

static void report(const char *name, float ms, int64_t arcs)
{
    printf("%-44s %8.3f ms  %7.1f G lookups/s  %6.2f TB/s at 5 B/arc\n", name, ms, arcs / ms * 1e-6, arcs * 5.0 / ms * 1e-9);
    fflush(stdout);
}

int main()
{
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int64_t arcs = (int64_t)1 << 29;
    const uint32_t slots = 196608;  // 192 KB of byte labels
    const uint32_t pslots = 245760; // 192 KB of 6-bit labels
    int32_t *t;
    uint8_t *tab, *cls;
    CK(cudaMalloc(&t, arcs * 4));
    CK(cudaMalloc(&cls, arcs));
    CK(cudaMalloc(&tab, 64 << 20));
    fill_table<<<1024, 256>>>(tab, 64 << 20);
    printf("SMs %d, arcs %lld\n", sms, (long long)arcs);

    fill_targets<<<sms * 8, 256>>>(t, arcs, slots);
    CK(cudaDeviceSynchronize());
    const int sh = 196608;
    CK(cudaFuncSetAttribute(k_tile_bytes<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh));
    CK(cudaFuncSetAttribute(k_tile_bytes<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh));
    CK(cudaFuncSetAttribute(k_tile_vec<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh));
    CK(cudaFuncSetAttribute(k_tile_vec<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh));
    CK(cudaFuncSetAttribute(k_tile_vec<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh));
    CK(cudaFuncSetAttribute(k_tile_packed<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh));
    report("stream only, v4 loads x4", time_ms([&] { k_stream_only<4><<<sms, 1024>>>(t, arcs, cls); }), arcs);
    report("stream only, v4 loads x2", time_ms([&] { k_stream_only<2><<<sms, 1024>>>(t, arcs, cls); }), arcs);
    report("smem byte tile, b32 loads x16, byte stores",
           time_ms([&] { k_tile_bytes<16><<<sms, 1024, sh>>>(t, arcs, tab, slots, cls); }), arcs);
    report("smem byte tile, b32 loads x8, byte stores",
           time_ms([&] { k_tile_bytes<8><<<sms, 1024, sh>>>(t, arcs, tab, slots, cls); }), arcs);
    report("smem byte tile, v4 loads x2, word stores",
           time_ms([&] { k_tile_vec<2><<<sms, 1024, sh>>>(t, arcs, tab, slots, cls); }), arcs);
    report("smem byte tile, v4 loads x4, word stores",
           time_ms([&] { k_tile_vec<4><<<sms, 1024, sh>>>(t, arcs, tab, slots, cls); }), arcs);
    report("smem byte tile, v4 loads x6, word stores",
           time_ms([&] { k_tile_vec<6><<<sms, 1024, sh>>>(t, arcs, tab, slots, cls); }), arcs);
    fill_targets<<<sms * 8, 256>>>(t, arcs, 98304);
    CK(cudaDeviceSynchronize());
    report("smem byte tile 96 KB, v4 loads x4",
           time_ms([&] { k_tile_vec<4><<<sms, 1024, 98304>>>(t, arcs, tab, 98304, cls); }), arcs);
    fill_targets<<<sms * 8, 256>>>(t, arcs, pslots);
    CK(cudaDeviceSynchronize());
    report("smem 6-bit tile, v4 loads x4, word stores",
           time_ms([&] { k_tile_packed<4><<<sms, 1024, sh>>>(t, arcs, tab, pslots, cls); }), arcs);
    for (uint32_t range : {16384u, 32768u, 65536u, 131072u, 1u << 20, 1u << 24}) {
        fill_targets<<<sms * 8, 256>>>(t, arcs, range);
        CK(cudaDeviceSynchronize());
        char name[96];
        snprintf(name, sizeof name, "global lookups over %u B (b32 x16)", range);
        report(name, time_ms([&] { k_global_lookup<16><<<sms, 1024>>>(t, arcs / 4, tab, cls); }), arcs / 4);
    }
    printf("done\n");
    return 0;
}
