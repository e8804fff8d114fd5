// Host driver for tests/test_lanesim_host.py: compiles the kernel's per-lane
// simulator (paper_1712_04495_b200/csrc/sgpu_lanesim.cuh, LaneSim) with the
// host C++ compiler and runs it on traces read from stdin, so the exact
// decision logic of K1 v5 is checked against the oracle without a GPU.
// Staging (arrival order, fit table, class masks) is rebuilt here from its
// definition in sgpu_lane.cu's stage_trace, single device.
//
// stdin, per case:  n policy cap keys  then n lines: arrival mem busy prio
//   keys: 1 = 32-bit keys, 0 = 64-bit keys with the main pass's heap
//   (kLaneHeapW), 2 = 64-bit keys with the retry pass's heap (kLaneHeapN)
// stdout, per case: ok T B I grants pops maxh unfinished  grant_0 end_0 ... (app order)
#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_1712_04495_b200/csrc/sgpu_lanesim.cuh"

using namespace sg;

template <int K, bool NAR, uint32_t HW = kLaneHeapW, bool TB = (K <= 4)>
static void run_case(int n, uint32_t policy, uint32_t cap, const std::vector<uint32_t>& A,
                     const std::vector<uint32_t>& M, const std::vector<uint32_t>& Bz,
                     const std::vector<uint32_t>& Pr) {
    constexpr uint32_t N = 32u * K;
    using Sim = LaneSim<K, NAR, HW, FitStride<K>::v, TB>;  // fit table stride FitStride<K>
    using PT = typename Sim::PT;
    constexpr uint32_t NW = Sim::NW;
    // arrival order: (arrival, index)
    std::vector<int> ord(n);
    for (int i = 0; i < n; i++) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return A[x] < A[y]; });
    std::vector<uint32_t> s_a(N + 4, 0), s_mem(N + 4, ~0u), s_bw(N + 4, 0);
    uint32_t z = 0;
    for (int e = 0; e < n; e++) {
        const int i = ord[e];
        s_a[e] = A[i];
        s_mem[e] = M[i];
        s_bw[e] = Bz[i] | ((uint32_t)i << kBusyBits);
        z += A[i] == 0;
    }
    // priority classes, highest first (policy.py:58-63)
    std::vector<uint32_t> pl;
    for (int e = 0; e < n; e++) pl.push_back(Pr[ord[e]]);
    std::sort(pl.begin(), pl.end());
    pl.erase(std::unique(pl.begin(), pl.end()), pl.end());
    std::reverse(pl.begin(), pl.end());
    if (pl.size() > kLaneMaxCls) { printf("0\n"); return; }
    std::vector<uint64_t> s_cm((pl.size() + 1) * NW, 0);
    for (size_t c = 0; c < pl.size(); c++)
        for (int e = 0; e < n; e++)
            if (Pr[ord[e]] == pl[c]) {
                s_cm[c * NW + (e >> 6)] |= 1ull << (e & 63);
                s_bw[e] |= (uint32_t)c << kClsShift;
            }
    // fit table: requests ascending, T at every 4th rank, rank -> position
    std::vector<int> rk(n);
    for (int e = 0; e < n; e++) rk[e] = e;
    std::stable_sort(rk.begin(), rk.end(), [&](int x, int y) { return s_mem[x] < s_mem[y]; });
    std::vector<PT> s_por(N + 16, (PT)N), s_lt(LtBuckets<FitStride<K>::v>::v + 16, 0);  // (host: roomier than the kernel slots)
    for (int r = 0; r < n; r++) s_por[r] = (PT)rk[r];
    const uint32_t mn = n ? s_mem[rk[0]] : 0, mx = n ? s_mem[rk[n - 1]] : 0;
    const uint64_t sc = ((uint64_t)LtBuckets<FitStride<K>::v>::v << 32) / ((uint64_t)(mx - mn) + 1);
    const uint32_t scale = sc > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)sc;
    for (uint32_t j = 0; j < LtBuckets<FitStride<K>::v>::v; j++) {  // first rank whose bucket is >= j
        uint32_t r = 0;
        while (r < (uint32_t)n && lt_bucket<FitStride<K>::v>(s_mem[rk[r]] - mn, scale) + 1 <= j) r++;
        s_lt[j] = (PT)r;
    }
    constexpr uint32_t FS = FitStride<K>::v;
    std::vector<uint64_t> s_t4((N / FS + 2) * NW, 0);
    uint64_t T[NW] = {};
    for (uint32_t r = 0; r < N; r++) {
        if (r < (uint32_t)n) T[rk[r] >> 6] |= 1ull << (rk[r] & 63);
        if ((r + 1) % FS == 0)
            for (uint32_t w = 0; w < NW; w++) s_t4[((r + 1) / FS) * NW + w] = T[w];
    }
    std::vector<uint64_t> heap(96 * 32, 0);  // column 0 of the [slot][lane] layout
    std::vector<uint32_t> grant(n, SG_NEVER), end(n, SG_NEVER);
    SimParams P{grant.data(), end.data()};
    Sim sim(P);
    sim.s_a = s_a.data();
    sim.s_mem = s_mem.data();
    sim.s_bw = s_bw.data();
    sim.s_por = s_por.data();
    sim.s_lt = s_lt.data();
    sim.lt_lo = mn;
    sim.lt_hi = mx;
    sim.lt_scale = scale;
    sim.s_t4 = s_t4.data();
    sim.s_cm = s_cm.data();
    sim.ncls = (uint32_t)pl.size();
    sim.heap = reinterpret_cast<typename Sim::Key*>(heap.data());
    sim.gp = grant.data();
    sim.ep = end.data();
    if (!sim.run((uint32_t)n, 0, (uint32_t)n, z, policy, cap)) { printf("0\n"); return; }
    uint32_t unf = 0;
    for (uint64_t bits = sim.mask[0]; bits; bits &= bits - 1) unf++;
    for (uint32_t w = 1; w < Sim::NW; w++)
        for (uint64_t bits = sim.mask[w]; bits; bits &= bits - 1) unf++;
    const uint64_t Iv = (sim.last == 0 && sim.used != 0)
                            ? (uint64_t)sim.used
                            : sim.I + (uint64_t)sim.used * (sim.last - sim.mem_t);
    printf("1 %u %u %llu %u %u %u %u", sim.last, sim.B, (unsigned long long)Iv, sim.grants,
           sim.pops + (uint32_t)n, sim.maxh, unf);
    for (int i = 0; i < n; i++) printf(" %u %u", grant[i], end[i]);
    printf("\n");
}

int main() {
    int n, narrow;
    unsigned policy, cap;
    while (scanf("%d %u %u %d", &n, &policy, &cap, &narrow) == 4) {
        std::vector<uint32_t> A(n), M(n), Bz(n), Pr(n);
        for (int i = 0; i < n; i++)
            if (scanf("%u %u %u %u", &A[i], &M[i], &Bz[i], &Pr[i]) != 4) return 1;
        if (n <= 32) {
            if (narrow == 1) run_case<1, true>(n, policy, cap, A, M, Bz, Pr);
            else if (narrow == 2) run_case<1, false, kLaneHeapN>(n, policy, cap, A, M, Bz, Pr);
            else run_case<1, false>(n, policy, cap, A, M, Bz, Pr);
        } else if (n <= 64) {
            if (narrow == 1) run_case<2, true>(n, policy, cap, A, M, Bz, Pr);
            else if (narrow == 2) run_case<2, false, kLaneHeapN>(n, policy, cap, A, M, Bz, Pr);
            else run_case<2, false>(n, policy, cap, A, M, Bz, Pr);
        } else if (n <= 128) {
            if (narrow == 1) run_case<4, true>(n, policy, cap, A, M, Bz, Pr);
            else if (narrow == 2) run_case<4, false, kLaneHeapN>(n, policy, cap, A, M, Bz, Pr);
            else run_case<4, false>(n, policy, cap, A, M, Bz, Pr);
        } else {
            // 256 apps: the global-table kernel's simulator (fit table, u16
            // rank tables, 32-key three-level heap) for both key widths
            if (narrow == 1) run_case<8, true, 32, true>(n, policy, cap, A, M, Bz, Pr);
            else run_case<8, false, 32, true>(n, policy, cap, A, M, Bz, Pr);
        }
        fflush(stdout);
    }
    return 0;
}
