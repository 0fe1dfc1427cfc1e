// Host memory bandwidth probe (dev tool): T threads write / read a buffer.
// g++ -O3 -march=x86-64-v3 -pthread tools/host_bw.cpp -o tools/host_bw
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <immintrin.h>
int main(int argc, char **argv)
{
    size_t gb = argc > 1 ? atol(argv[1]) : 8;
    int T = argc > 2 ? atoi(argv[2]) : (int)std::thread::hardware_concurrency();
    size_t n = gb << 30;
    char *buf = (char *)aligned_alloc(64, n);
    memset(buf, 1, n);
    auto run = [&](const char *name, auto fn) {
        for (int rep = 0; rep < 3; rep++) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; t++) th.emplace_back([&, t] { fn(buf + n / T * t, n / T); });
            for (auto &x : th) x.join();
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            printf("%s threads=%d %.1f GB/s\n", name, T, n / s / 1e9);
        }
    };
    run("memset", [](char *p, size_t m) { memset(p, 0, m); });
    run("stream_store", [](char *p, size_t m) {
        __m256i z = _mm256_setzero_si256();
        for (size_t i = 0; i + 32 <= m; i += 32) _mm256_stream_si256((__m256i *)(p + i), z);
        _mm_sfence();
    });
    volatile long sink = 0;
    run("read", [&](char *p, size_t m) {
        long s = 0;
        for (size_t i = 0; i < m; i += 64) s += p[i];
        sink += s;
    });
    return 0;
}
