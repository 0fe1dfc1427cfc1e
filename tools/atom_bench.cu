// Shared-memory atomic lane rate by address pattern (dev tool): random
// addresses (bank conflicts ~3.5-way), conflict-free (bank = lane), and
// conflict-free fire-and-forget u32 pairs (the weighted reducers' two planes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/atom_bench tools/atom_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void k_atom(int iters, unsigned long long *sink)
{
    __shared__ uint32_t s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t h = mix(threadIdx.x + blockIdx.x * 977);
    for (int i = 0; i < iters; i++) {
        h = h * 1664525u + 1013904223u;
        const uint32_t a = h >> 19;
        if (MODE == 0) atomicAdd(&s[a], h & 15u);                          // random
        if (MODE == 1) atomicAdd(&s[(a & ~31u) | lane], h & 15u);          // bank = lane
        if (MODE == 2) atomicAdd(&s[((a & 63u) << 5) | lane], h & 15u);    // [class][lane], 64 classes
        if (MODE == 3) {                                                  // plain RMW, bank = lane
            uint32_t *p = &s[((a & 63u) << 5) | lane];
            *p += h & 15u;
        }
        if (MODE == 4) atomicAdd(&s[a & ~1023u | ((a & 63u) * 56 + 3) % 1024], h & 15u);  // window-like: slot*56+class
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)s[5]);
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *sink;
    cudaMalloc(&sink, 8);
    const char *names[] = {"random", "bank = lane", "[class][lane]", "plain RMW [class][lane]", "window-like"};
    for (int mode = 0; mode < 5; mode++) {
        for (int per = 2; per <= 4; per += 2) {
            auto k = mode == 0 ? k_atom<0> : mode == 1 ? k_atom<1> : mode == 2 ? k_atom<2> : mode == 3 ? k_atom<3> : k_atom<4>;
            const int iters = 4096;
            k<<<sms * per, 256>>>(iters, sink);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            k<<<sms * per, 256>>>(iters, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double ops = (double)sms * per * 256 * iters;
            printf("%-26s %d CTA/SM: %.2f lane-ops/clk/SM (1.9 GHz)\n", names[mode], per, ops / (ms * 1e-3) / sms / 1.9e9);
        }
    }
    return 0;
}
