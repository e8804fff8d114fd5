// Host-side probe for the e2e pipeline design (run on the GPU box):
// device -> host copy of packed 16-bit (grant, end) tick pairs through a
// small ring of pinned staging slots, expanded by host threads into the
// caller's two u32 arrays with streaming stores, while the 1 GiB input
// streams host -> device on another stream (C2: 64M apps x 4 policies).
// The question: does a ring small enough to stay in the LLC cut host DRAM
// traffic (DMA write + re-read) against staging through DRAM?
//   nvcc -O3 -std=c++17 -Xcompiler -mavx2 -o /tmp/ring profiles/ring_probe.cu && /tmp/ring
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// expand n (grant16, end16) pairs: 0xFFFF -> 0xFFFFFFFF
__attribute__((target("avx2"))) static void expand(const uint16_t* src, uint32_t* g, uint32_t* e, uint64_t n) {
    const __m256i ff = _mm256_set1_epi32(0xFFFF);
    uint64_t i = 0;
    for (; i + 8 <= n; i += 8) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 2 * i));
        __m256i lo = _mm256_and_si256(v, ff);
        __m256i hi = _mm256_srli_epi32(v, 16);
        lo = _mm256_or_si256(lo, _mm256_slli_epi32(_mm256_cmpeq_epi32(lo, ff), 16));
        hi = _mm256_or_si256(hi, _mm256_slli_epi32(_mm256_cmpeq_epi32(hi, ff), 16));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(g + i), lo);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(e + i), hi);
    }
    for (; i < n; i++) {
        const uint32_t a = src[2 * i], b = src[2 * i + 1];
        g[i] = a == 0xFFFF ? 0xFFFFFFFFu : a;
        e[i] = b == 0xFFFF ? 0xFFFFFFFFu : b;
    }
}

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const uint64_t PAIRS = 64ull << 20 << 2;   // 64M apps x 4 policies
    const uint64_t in_b = 1ull << 30;
    uint8_t *h_in, *d_in;
    uint16_t* d_src;
    CK(cudaMallocHost(&h_in, in_b));
    CK(cudaMalloc(&d_in, in_b));
    CK(cudaMalloc(&d_src, PAIRS * 4));
    CK(cudaMemset(d_src, 1, PAIRS * 4));
    memset(h_in, 1, in_b);
    uint32_t *g, *e;
    CK(cudaMallocHost(&g, PAIRS * 4));
    CK(cudaMallocHost(&e, PAIRS * 4));
    memset(g, 0, PAIRS * 4);
    memset(e, 0, PAIRS * 4);
    cudaStream_t s_in, s_out;
    CK(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    const int nthr = argc > 1 ? atoi(argv[1]) : 15;

    // PCIe alone
    for (int rep = 0; rep < 2; rep++) {
        double t0 = now();
        CK(cudaMemcpyAsync(d_in, h_in, in_b, cudaMemcpyHostToDevice, s_in));
        CK(cudaStreamSynchronize(s_in));
        double t1 = now();
        CK(cudaMemcpyAsync(g, d_src, PAIRS * 4, cudaMemcpyDeviceToHost, s_out));
        CK(cudaStreamSynchronize(s_out));
        double t2 = now();
        CK(cudaMemcpyAsync(d_in, h_in, in_b, cudaMemcpyHostToDevice, s_in));
        CK(cudaMemcpyAsync(g, d_src, PAIRS * 4, cudaMemcpyDeviceToHost, s_out));
        CK(cudaStreamSynchronize(s_in));
        CK(cudaStreamSynchronize(s_out));
        double t3 = now();
        printf("pcie: h2d 1 GiB %.1f ms (%.1f GB/s), d2h 1 GiB %.1f ms (%.1f GB/s), both %.1f ms\n",
               (t1 - t0) * 1e3, in_b / (t1 - t0) / 1e9, (t2 - t1) * 1e3, PAIRS * 4 / (t2 - t1) / 1e9, (t3 - t2) * 1e3);
    }
    // host expand alone (source in DRAM)
    {
        uint16_t* big;
        CK(cudaMallocHost(&big, PAIRS * 4));
        memset(big, 3, PAIRS * 4);
        for (int rep = 0; rep < 2; rep++) {
            double t0 = now();
            std::vector<std::thread> th;
            for (int w = 0; w < nthr; w++)
                th.emplace_back([&, w]() {
                    const uint64_t lo = PAIRS * w / nthr & ~15ull, hi = w + 1 == nthr ? PAIRS : PAIRS * (w + 1) / nthr & ~15ull;
                    expand(big + 2 * lo, g + lo, e + lo, hi - lo);
                    _mm_sfence();
                });
            for (auto& t : th) t.join();
            double t1 = now();
            printf("expand from DRAM, %d threads: %.1f ms (%.1f GB/s r+w)\n", nthr, (t1 - t0) * 1e3,
                   PAIRS * 12 / (t1 - t0) / 1e9);
        }
        cudaFreeHost(big);
    }
    // ring v2: slot k is expanded by thread k % nthr alone (no per-slot
    // split, no cross-thread counters on the slot), R = slots_per_thread *
    // nthr; optionally a fraction of the policies copied directly as u32
    // grant + end into the final arrays (PCIe 8 B, host DRAM 8 B per app-
    // policy) instead of packed 16-bit pairs through the ring
    const uint64_t slot_sizes[] = {512u << 10, 1u << 20, 2u << 20};
    const int per_thr[] = {2, 4};
    const double directs[] = {0.0, 0.25};
    for (double fdir : directs)
    for (uint64_t S : slot_sizes) {
        for (int spt : per_thr) {
            const int R = spt * nthr;
            uint8_t* ring;
            CK(cudaMallocHost(&ring, R * S));
            memset(ring, 0, R * S);
            std::vector<cudaEvent_t> ev(R);
            for (auto& x : ev) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
            const uint64_t dir_pairs = (uint64_t)(PAIRS * fdir) & ~((S / 4) - 1);
            const uint64_t ring_pairs = PAIRS - dir_pairs;
            const uint64_t nchunks = ring_pairs * 4 / S;
            const uint64_t pairs_per = S / 4;
            cudaStream_t s_dir;
            CK(cudaStreamCreateWithFlags(&s_dir, cudaStreamNonBlocking));
            for (int rep = 0; rep < 2; rep++) {
                std::vector<std::atomic<int64_t>> freed(R), issued(R);
                for (int i = 0; i < R; i++) { freed[i] = -1; issued[i] = -1; }
                double t0 = now();
                CK(cudaMemcpyAsync(d_in, h_in, in_b, cudaMemcpyHostToDevice, s_in));
                if (dir_pairs) {  // u32 grant + end of the direct policies (sources: any device bytes)
                    CK(cudaMemcpyAsync(g + ring_pairs, d_src, dir_pairs * 4, cudaMemcpyDeviceToHost, s_dir));
                    CK(cudaMemcpyAsync(e + ring_pairs, d_src, dir_pairs * 4, cudaMemcpyDeviceToHost, s_dir));
                }
                std::thread coord([&]() {
                    for (uint64_t k = 0; k < nchunks; k++) {
                        const int s = (int)(k % R);
                        // the slot's previous chunk (k - R) must be expanded
                        while (k >= (uint64_t)R && freed[s].load(std::memory_order_acquire) != (int64_t)(k - R)) _mm_pause();
                        CK(cudaMemcpyAsync(ring + s * S, reinterpret_cast<uint8_t*>(d_src) + k * S, S,
                                           cudaMemcpyDeviceToHost, s_out));
                        CK(cudaEventRecord(ev[s], s_out));
                        issued[s].store((int64_t)k, std::memory_order_release);
                    }
                });
                std::vector<std::thread> th;
                for (int w = 0; w < nthr; w++)
                    th.emplace_back([&, w]() {
                        for (uint64_t k = w; k < nchunks; k += nthr) {
                            const int s = (int)(k % R);
                            while (issued[s].load(std::memory_order_acquire) != (int64_t)k) _mm_pause();
                            CK(cudaEventSynchronize(ev[s]));
                            const uint64_t base = k * pairs_per;
                            expand(reinterpret_cast<const uint16_t*>(ring + s * S), g + base, e + base, pairs_per);
                            freed[s].store((int64_t)k, std::memory_order_release);
                        }
                        _mm_sfence();
                    });
                coord.join();
                for (auto& t : th) t.join();
                CK(cudaStreamSynchronize(s_in));
                CK(cudaStreamSynchronize(s_dir));
                double t1 = now();
                if (rep == 1)
                    printf("ring2 S=%5.2f MB R=%2d (%.0f MB) direct %.2f, %d threads + 1 GiB h2d: %.1f ms\n",
                           S / 1048576.0, R, R * S / 1048576.0, fdir, nthr, (t1 - t0) * 1e3);
            }
            cudaStreamDestroy(s_dir);
            for (auto& x : ev) cudaEventDestroy(x);
            cudaFreeHost(ring);
        }
    }
    return 0;
}
