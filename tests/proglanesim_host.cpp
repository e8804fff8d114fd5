// Host driver for tests/test_proglanesim_host.py: compiles the step-program
// lane simulator (paper_1712_04495_b200/csrc/sgpu_proglanesim.cuh,
// ProgLaneSim) with the host C++ compiler and runs it on step programs read
// from stdin, so the kernel's decision logic is checked against the oracle
// without a GPU.  The slot staging (packed steps, first-step indices,
// priority ranks) is rebuilt here as sgpu_proglane.cu's prog_stage does.
//
// stdin, per case:  n policy cap nsteps
//                   n + 1 lines: first-step index per app (relative), last = nsteps
//                   n lines: priority rank
//                   nsteps lines: op mib dur
// stdout, per case: ok T B I grants pops maxh unfinished  grant_0 end_0 ... (app order)
#include <cstdio>
#include <vector>

#include "../paper_1712_04495_b200/csrc/sgpu_proglanesim.cuh"

using namespace sg;

template <int NA>
static void run_case(uint32_t n, uint32_t policy, uint32_t cap, const std::vector<uint16_t>& first,
                     const std::vector<uint8_t>& prio, const std::vector<uint64_t>& st) {
    constexpr uint32_t HS = ProgLaneSim<NA>::HS;
    std::vector<uint64_t> heap(NA * HS, 0);
    std::vector<uint16_t> pc(NA * HS, 0);
    std::vector<int32_t> held(NA * HS, 0);
    std::vector<uint8_t> q(NA * HS, 0);
    std::vector<uint32_t> grant(n, SG_NEVER), end(n, SG_NEVER);
    ProgLaneSim<NA> sim(ProgHostOut{grant.data(), end.data()});
    sim.st = st.data();
    sim.first = first.data();
    sim.prio = prio.data();
    sim.heap = heap.data();
    sim.pc = pc.data();
    sim.held = held.data();
    sim.q = q.data();
    sim.out_base = 0;
    if (!sim.run(n, policy, cap)) { printf("0\n"); return; }
    uint32_t unf = 0;
    for (uint32_t a = 0; a < n; a++) unf += !((sim.ended >> a) & 1u);
    // makespan T, busy B, memory integral I with the final level term
    const uint64_t Iv = (sim.last == 0 && sim.used != 0)
                            ? (uint64_t)sim.used
                            : sim.I + (uint64_t)(sim.used * (int64_t)(sim.last - sim.mem_t));
    printf("1 %u %u %llu %u %u %u %u", sim.last, sim.B, (unsigned long long)Iv, sim.grants,
           sim.pops + n, sim.maxh, unf);
    for (uint32_t i = 0; i < n; i++) printf(" %u %u", grant[i], end[i]);
    printf("\n");
}

int main() {
    unsigned n, policy, cap, ns;
    while (scanf("%u %u %u %u", &n, &policy, &cap, &ns) == 4) {
        std::vector<uint16_t> first(n + 1);
        std::vector<uint8_t> prio(n + 1, 0);
        std::vector<uint64_t> st(ns + 1, 0);
        for (unsigned i = 0; i <= n; i++) { unsigned v; if (scanf("%u", &v) != 1) return 1; first[i] = (uint16_t)v; }
        for (unsigned i = 0; i < n; i++) { unsigned v; if (scanf("%u", &v) != 1) return 1; prio[i] = (uint8_t)v; }
        for (unsigned j = 0; j < ns; j++) {
            unsigned op, mib;
            unsigned long long dur;
            if (scanf("%u %u %llu", &op, &mib, &dur) != 3) return 1;
            st[j] = pack_step(op, mib, dur);
        }
        if (n <= 16) run_case<16>(n, policy, cap, first, prio, st);
        else run_case<32>(n, policy, cap, first, prio, st);
        fflush(stdout);
    }
    return 0;
}
