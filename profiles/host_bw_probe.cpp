// Host-memory probe for the e2e pipeline (run on the GPU box): derive grants (grant = end - busy)
// for 1M traces x 64 apps x 4 policies with N threads, and a threaded memcpy of 1.07 GB.
//   g++ -O3 -std=c++17 -pthread -o /tmp/hbw profiles/host_bw_probe.cpp && /tmp/hbw 16
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cstdlib>
struct App { uint32_t a, mem, busy, attr; };
__attribute__((target("avx2"))) void row(const uint32_t* mem, const uint32_t* busy, const uint32_t* e, uint32_t* g, uint32_t n) {
    const __m256i never = _mm256_set1_epi32(-1), zero = _mm256_setzero_si256();
    for (uint32_t i = 0; i + 8 <= n; i += 8) {
        __m256i ev = _mm256_loadu_si256((const __m256i*)(e + i)), mv = _mm256_loadu_si256((const __m256i*)(mem + i)), bv = _mm256_loadu_si256((const __m256i*)(busy + i));
        __m256i no = _mm256_or_si256(_mm256_cmpeq_epi32(mv, zero), _mm256_cmpeq_epi32(ev, never));
        _mm256_stream_si256((__m256i*)(g + i), _mm256_blendv_epi8(_mm256_sub_epi32(ev, bv), never, no));
    }
}
int main(int argc, char** argv) {
    const uint64_t NT = 1 << 20, NA = 64, NP = 4, TOT = NT * NA;
    int nthr = argc > 1 ? atoi(argv[1]) : 16;
    App* apps = (App*)aligned_alloc(64, TOT * 16);
    uint32_t* end = (uint32_t*)aligned_alloc(64, TOT * NP * 4);
    uint32_t* grant = (uint32_t*)aligned_alloc(64, TOT * NP * 4);
    uint32_t* dst = (uint32_t*)aligned_alloc(64, TOT * NP * 4);
    memset(apps, 1, TOT * 16); memset(end, 2, TOT * NP * 4); memset(grant, 0, TOT * NP * 4); memset(dst, 0, TOT * NP * 4);
    for (int rep = 0; rep < 3; rep++) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int w = 0; w < nthr; w++) th.emplace_back([&, w]() {
            uint32_t mem[64], busy[64];
            for (uint64_t t = NT * w / nthr; t < NT * (w + 1) / nthr; t++) {
                for (int i = 0; i < 64; i++) { mem[i] = apps[t * 64 + i].mem; busy[i] = apps[t * 64 + i].busy; }
                for (uint64_t p = 0; p < NP; p++) row(mem, busy, end + p * TOT + t * 64, grant + p * TOT + t * 64, 64);
            }
            _mm_sfence();
        });
        for (auto& x : th) x.join();
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        auto t1 = std::chrono::steady_clock::now();
        std::vector<std::thread> th2;
        for (int w = 0; w < nthr; w++) th2.emplace_back([&, w]() {
            uint64_t lo = TOT * NP * w / nthr, hi = TOT * NP * (w + 1) / nthr;
            memcpy(dst + lo, end + lo, (hi - lo) * 4);
        });
        for (auto& x : th2) x.join();
        double dt2 = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
        printf("threads %d: derive %.1f ms (%.1f GB/s moved)  memcpy 1.07 GB %.1f ms (%.1f GB/s r+w)\n", nthr, dt * 1e3, (TOT * 16 + 2 * TOT * NP * 4) / dt / 1e9, dt2 * 1e3, 2 * TOT * NP * 4 / dt2 / 1e9);
    }
}
