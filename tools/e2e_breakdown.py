"""Where the end-to-end time of run_saw_pool goes (C4 workload, one B200)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_07222_b200 as labs  # noqa: E402

cfg = labs.SawConfig(length=451, walkers=1024, prefix_len=8, target_merit=5.3, max_restarts=64, seed=1)
labs.run_saw_pool(cfg, labs.CollectingSink())
for label, mk in [("no sink", lambda: None), ("CollectingSink", labs.CollectingSink),
                  ("CollectingSink+take", labs.CollectingSink)]:
    ts = []
    for _ in range(3):
        sink = mk()
        t0 = time.perf_counter()
        st = labs.run_saw_pool(cfg, sink)
        if label.endswith("take"):
            sink.take()
        ts.append(time.perf_counter() - t0)
    print(f"{label:22s} wall {min(ts) * 1e3:8.1f} ms  pool wall {st.wall_seconds * 1e3:8.1f} ms  "
          f"kernel {st.kernel_ms:7.1f} ms  seed {st.seed_ms:5.2f} ms  d2h {st.d2h_bytes / 1e6:.1f} MB")
