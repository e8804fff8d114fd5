// sgpu_proglanesim.cuh — the per-lane simulation of K1 v6 (ProgLaneSim): one
// (trace, policy) of a STEP-PROGRAM trace simulated by one thread, from a
// staged trace slot.  The reference's general workload shape: every app is
// an AppProfile of several phases (memshare/harness.py:39-83), flattened to
// cpu / alloc / busy / free steps (harness.py:478-490); apps may hold memory
// across cpu steps, allocate several times, and wait in the queue more than
// once.  Included by sgpu_proglane.cu (device) and, with the shims below,
// compiled by the host C++ compiler for tests/test_proglanesim_host.py, which
// checks this decision logic against the oracle on CPU.
//
// Restated from the reference, one lane per simulation:
//   * event order: the (t, push counter) heap of harness.py:505-508,563-565
//     as a per-lane 4-ary heap of 64-bit keys t << 32 | counter << AB | app
//     in shared memory ([slot][lane] layout); every app has at most one
//     pending entry, so the heap holds at most n keys.  The initial pops
//     (harness.py:560-562: all apps at t = 0, counters 1..n, before any
//     later push) run in index order before the heap loop.
//   * advance (harness.py:510-543): cpu / busy push (now + d, ++counter);
//     alloc takes free memory at once (the arrival bypass, 521-531) or
//     enqueues; free releases, runs grant_waiters and continues.
//   * grant_waiters (harness.py:545-558) + select_grants (policy.py:52-74):
//     the wait queue is a per-lane list of app ids in enqueue order; a round
//     scans it once with a shrinking budget (FIFO stops at the first misfit
//     of the round's class, MMU skips it; the priority kinds restrict to the
//     top waiting priority), applies each grant in queue order (push (now,
//     ++counter)) and compacts the list; priority kinds repeat while the
//     round granted (the next class is served in the same tick).
//   * statistics: harness.py:373-461 integer forms accumulated at pop time,
//     as TraceSim's program mode (sgpu_tracesim.cuh) does, so the record of
//     both engines is identical by construction.
// A lane fails (and its simulation is re-run by the warp engine) when an
// event time would pass 2^32 - 2 ticks or the push counter its key field.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#include "sgpu_tracesim.cuh"
#define SG_PHD __device__ __forceinline__
#else
#include <algorithm>
#include "../../include/sgpu.h"
#define SG_PHD inline
namespace sg {
using std::max;
using std::min;
struct ProgHostOut {  // the two output arrays ProgLaneSim writes
    uint32_t* grant;
    uint32_t* end;
};
}  // namespace sg
#endif

namespace sg {

constexpr uint32_t kStepValBits = 62;  // packed step: op << 62 | value
constexpr uint64_t kStepValMask = (1ull << kStepValBits) - 1ull;
constexpr uint32_t kPcBusy = 0x8000u;  // pc bit: the pending pop ends a busy step

SG_PHD uint64_t pack_step(uint32_t op, uint32_t mib, uint64_t dur) {
    op = op <= SG_OP_FREE ? op : SG_OP_FREE;  // the warp engine runs any other op as a free
    const uint64_t v = (op == SG_OP_CPU || op == SG_OP_BUSY) ? (dur < kStepValMask ? dur : kStepValMask) : mib;
    return ((uint64_t)op << kStepValBits) | v;
}

// NA: apps per trace slot (16 or 32); AB: app bits of a heap key.
template <int NA> struct ProgLaneSim {
    static constexpr uint32_t AB = NA <= 16 ? 4u : 5u;
    static constexpr uint32_t CLIM = 1u << (32u - AB);  // push counters stay below
    static constexpr uint32_t HS = 32;                   // column stride ([slot][lane] layout)

#ifdef __CUDACC__
    const SimParams& P;
    SG_PHD ProgLaneSim(const SimParams& p) : P(p) {}
#else
    ProgHostOut P;
    ProgLaneSim(ProgHostOut p) : P(p) {}
#endif
    // slot (shared by the trace's lanes)
    const uint64_t* st;      // packed steps of the trace
    const uint16_t* first;   // first step of app i (n + 1 entries)
    const uint8_t* prio;     // priority rank of app i
    // this lane's columns
    uint64_t* heap;          // heap[h * HS]
    uint16_t* pc;            // pc[a * HS] (| kPcBusy)
    int32_t* held;           // held[a * HS]: the app's allocated MiB (harness.py:401-406)
    uint8_t* q;              // q[k * HS]: waiting apps in enqueue order
    uint64_t out_base;       // grant/end index of app 0 of the trace under this policy
    uint32_t n, cap;
    bool prio_pol, mmu, fail;
    uint32_t hs, qlen, counter;
    uint32_t granted, ended;  // bit a: first grant written / end emitted
    int64_t used;
    // statistics (harness.py:373-461 integer forms)
    uint32_t last, mem_t, busy_prev, B;
    uint64_t I;
    int32_t busy_level, holders;
    uint32_t maxh, grants, pops;

    SG_PHD void mem_point(uint32_t now) {
        I += (uint64_t)(used * (int64_t)(now - mem_t));
        mem_t = now;
    }
    SG_PHD void busy_point(uint32_t now, int32_t delta) {
        B += busy_level > 0 ? now - busy_prev : 0u;
        busy_prev = now;
        busy_level += delta;
    }
    SG_PHD void out_grant(uint32_t a, uint32_t t) { reinterpret_cast<uint32_t*>(P.grant)[out_base + a] = t; }
    SG_PHD void out_end(uint32_t a, uint32_t t) { reinterpret_cast<uint32_t*>(P.end)[out_base + a] = t; }

    // ------------------------------------------------- event heap
    SG_PHD void push(uint64_t t, uint32_t a) {
        counter += 1;  // harness.py:505-508
        if (t > 0xFFFFFFFEull || counter >= CLIM) { fail = true; return; }
        const uint64_t key = (t << 32) | ((uint64_t)counter << AB) | a;
        uint32_t i = hs++;
        while (i > 0) {
            const uint32_t p = (i - 1u) >> 2;
            const uint64_t kp = heap[p * HS];
            if (key >= kp) break;
            heap[i * HS] = kp;
            i = p;
        }
        heap[i * HS] = key;
    }
    SG_PHD uint64_t pop() {
        const uint64_t top = heap[0];
        hs -= 1;
        const uint64_t lk = heap[hs * HS];
        uint32_t i = 0;
        while (true) {
            const uint32_t c = 4u * i + 1u;
            if (c >= hs) break;
            uint32_t m = c;
            uint64_t km = heap[c * HS];
            for (uint32_t j = 1; j < 4; j++) {
                if (c + j < hs) {
                    const uint64_t k = heap[(c + j) * HS];
                    if (k < km) { km = k; m = c + j; }
                }
            }
            if (km >= lk) break;
            heap[i * HS] = km;
            i = m;
        }
        heap[i * HS] = lk;
        return top;
    }

    SG_PHD void take(uint32_t a, uint32_t mib, int32_t& h, uint32_t now) {
        if (h <= 0 && h + (int32_t)mib > 0) holders += 1;
        h += (int32_t)mib;
        grants += 1;
        if (!((granted >> a) & 1u)) {  // first grant (the per-app output)
            granted |= 1u << a;
            out_grant(a, now);
        }
    }

    // grant_waiters (harness.py:545-558) + select_grants (policy.py:52-74)
    SG_PHD void grant_waiters(uint32_t now) {
        while (qlen > 0) {
            int64_t budget = (int64_t)cap - used;
            uint32_t top = 0;
            if (prio_pol)
                for (uint32_t k = 0; k < qlen; k++) top = max(top, (uint32_t)prio[q[k * HS]]);
            uint32_t removed = 0;
            bool stop = false;
            for (uint32_t k = 0; k < qlen; k++) {
                const uint32_t a = q[k * HS];
                bool g = false;
                uint32_t mib = 0;
                if (!stop && (!prio_pol || prio[a] == top)) {
                    const uint32_t p = pc[a * HS] & ~kPcBusy;
                    mib = (uint32_t)(st[first[a] + p] & kStepValMask);
                    mib = mib < 0x7FFFFFFFu ? mib : 0x7FFFFFFFu;  // the warp engine's saturated queue size
                    if ((int64_t)mib <= budget) {
                        g = true;
                        budget -= mib;
                    } else if (!mmu) {
                        stop = true;  // FIFO: a misfit blocks the rest of the class
                    }
                }
                if (g) {
                    // the grant in queue order: alloc, pc past the alloc, push (now, ++counter)
                    mem_point(now);
                    used += mib;
                    int32_t h = held[a * HS];
                    take(a, mib, h, now);
                    held[a * HS] = h;
                    pc[a * HS] = (uint16_t)(pc[a * HS] + 1u);
                    push(now, a);
                    removed += 1;
                } else if (removed) {
                    q[(k - removed) * HS] = (uint8_t)a;
                }
            }
            qlen -= removed;
            maxh = max(maxh, (uint32_t)max(holders, 0));
            // FIFO / MMU: a second round is provably empty; the priority kinds
            // serve the next class when the top one drained
            if (removed == 0 || !prio_pol) return;
        }
    }

    // harness.py:510-543
    SG_PHD void advance(uint32_t a, uint32_t now) {
        last = now;
        uint32_t p = pc[a * HS];
        int32_t h = held[a * HS];
        if (p & kPcBusy) {
            busy_point(now, -1);
            p &= ~kPcBusy;
        }
        const uint32_t f0 = first[a], len = first[a + 1] - f0;
        while (true) {
            if (p >= len) {  // end (harness.py:543)
                ended |= 1u << a;
                out_end(a, now);
                break;
            }
            const uint64_t s = st[f0 + p];
            const uint32_t op = (uint32_t)(s >> kStepValBits);
            const uint64_t v = s & kStepValMask;
            if (op == SG_OP_CPU || op == SG_OP_BUSY) {  // harness.py:514-520
                p += 1;
                if (op == SG_OP_BUSY) {
                    busy_point(now, +1);
                    p |= kPcBusy;
                }
                push((uint64_t)now + v, a);
                break;
            }
            const uint32_t mib = (uint32_t)v;
            if (op == SG_OP_ALLOC) {  // harness.py:521-536
                if (used + (int64_t)mib <= (int64_t)cap) {
                    mem_point(now);
                    used += mib;
                    take(a, mib, h, now);
                    maxh = max(maxh, (uint32_t)max(holders, 0));
                    p += 1;
                    continue;
                }
                q[qlen * HS] = (uint8_t)a;
                qlen += 1;
                break;
            }
            // free (harness.py:537-542)
            mem_point(now);
            used -= mib;
            if (h > 0 && h - (int32_t)mib <= 0) holders -= 1;
            h -= (int32_t)mib;
            p += 1;
            pc[a * HS] = (uint16_t)p;
            held[a * HS] = h;
            grant_waiters(now);
        }
        pc[a * HS] = (uint16_t)p;
        held[a * HS] = h;
    }

    // Simulate the slot's n apps under `policy`.  Returns false if the lane
    // must be re-run by the warp engine.
    SG_PHD bool run(uint32_t n_apps, uint32_t policy, uint32_t cap_mib) {
        n = n_apps;
        cap = cap_mib;
        prio_pol = policy >= SG_POLICY_PFIFO;
        mmu = (policy & 1u) != 0;
        fail = false;
        hs = qlen = 0;
        counter = n;  // the initial pushes took counters 1..n (harness.py:560-562)
        granted = ended = 0;
        used = 0;
        last = mem_t = busy_prev = B = 0;
        I = 0;
        busy_level = holders = 0;
        maxh = grants = pops = 0;
        for (uint32_t a = 0; a < n; a++) {
            pc[a * HS] = 0;
            held[a * HS] = 0;
        }
        for (uint32_t a = 0; a < n && !fail; a++) advance(a, 0u);
        while (hs > 0 && !fail) {  // harness.py:563-565
            const uint64_t k = pop();
            pops += 1;
            advance((uint32_t)k & ((1u << AB) - 1u), (uint32_t)(k >> 32));
        }
        return !fail;
    }

#ifdef __CUDACC__
    SG_PHD void finish(uint64_t rec, uint64_t seq) {
        const uint32_t all = n >= 32 ? ~0u : (1u << n) - 1u;
        for (uint32_t m = all & ~granted; m; m &= m - 1) out_grant((uint32_t)__ffs((int)m) - 1u, SG_NEVER);
        for (uint32_t m = all & ~ended; m; m &= m - 1) out_end((uint32_t)__ffs((int)m) - 1u, SG_NEVER);
        const uint32_t unf = n - (uint32_t)__popc(ended & all);
        store_tick_record(P, rec, n, cap, last, mem_t, I, B, used, grants, pops + n, maxh, unf, 0u, seq);
    }
#endif
};

}  // namespace sg
