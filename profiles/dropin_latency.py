"""Latency of the drop-in `simulate(spec)` (one workload per call) against
the reference's own `memshare.harness.simulate` (oracle/_ref) on the same
specs, one core.  Median of many calls after warm-up.

    python profiles/dropin_latency.py          (needs a GPU)
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import memshare.harness as RH  # noqa: E402

import paper_1712_04495_b200 as S  # noqa: E402


def med(fn, reps=200):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts) * 1e3


def main():
    cases = {
        "12 x ara-like": ([("ara-like", 12)], {}),
        "12 x mummer-like": ([("mummer-like", 12)], {}),
        "4+4+4 mixed @2400 pmmu": ([("ara-like", 4), ("mummer-like", 4), ("blast-like", 4)],
                                   {"policy": "pmmu", "device": {"devices": [{"mib": 2400}]}}),
    }
    for name, (inst, extra) in cases.items():
        doc = {"instances": [list(x) for x in inst], **extra}
        ours = S.WorkloadSpec.from_json(doc)
        ref = RH.WorkloadSpec.from_json(doc)
        a = S.simulate(ours)
        r = RH.simulate(ref)
        assert a.summary() == r.summary() and a.events == r.events and a.mem_trace == r.mem_trace
        t_ours = med(lambda: S.simulate(ours))
        t_ref = med(lambda: RH.simulate(ref))
        t_enc = med(lambda: S.harness.encode_spec(ours))
        enc = S.harness.encode_spec(ours)
        t_gpu = med(lambda: S.harness.run_encoded(enc, ours.policy))
        print(f"{name:24s} drop-in {t_ours:.3f} ms (encode {t_enc:.3f}, GPU call {t_gpu:.3f}, "
              f"report {t_ours - t_enc - t_gpu:.3f})  reference {t_ref:.3f} ms  "
              f"events {len(a.events)}  identical report")


if __name__ == "__main__":
    main()
