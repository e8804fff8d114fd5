"""Time repeated host-buffer pipeline calls (sg_simulate_batch_host) on C2
to see call-to-call variance, the chunk-size trade-off, and what the
per-app tick outputs cost (grant+end / end only / statistics only)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1712_04495_b200 import batch as B  # noqa: E402
from paper_1712_04495_b200.policy import policy_mask  # noqa: E402
from paper_1712_04495_b200.tracegen import CONFIGS  # noqa: E402

cfg = CONFIGS["C2"]
n, napp = cfg.n_traces, cfg.gen.apps_per_trace
_, pols = policy_mask(cfg.policies)
apps = B.generate_traces(cfg.gen, 0, n, device=0)
host = B.pinned_apps(n, napp)
host[...] = apps.cpu().numpy().view(np.uint32)
for variant in ("grant+end", "end", "stats"):
    outb = B.HostBuffers(len(pols), n, napp, cfg.ndev)
    if variant == "end":
        outb.grant = None
    if variant == "stats":
        outb.grant = outb.end = None
    for chunk in [int(x) for x in sys.argv[1:]] or [65536]:
        ts = []
        for i in range(5):
            t = time.perf_counter()
            B.simulate_batch_host(host, pols, cfg.cap_mib, device=0, out=outb, chunk_traces=chunk)
            ts.append(time.perf_counter() - t)
        print(f"{variant:10s} chunk {chunk}: " + " ".join(f"{x * 1e3:.1f}" for x in ts) + " ms/step; best "
              f"{n * len(pols) / min(ts):.3e} trace-sims/s")
