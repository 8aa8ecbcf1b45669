import time, sys
sys.path.insert(0,'.')
import paper_2409_07222_b200 as labs
for th in (16, 1):
    cfg = labs.SawConfig(length=101, walkers=64, prefix_len=8, target_merit=3.2, max_restarts=0, time_budget_s=0.5, seed=7, threads=th)
    sink = labs.CollectingSink()
    t0=time.time(); st=labs.run_saw_pool(cfg, sink); print(th, time.time()-t0, st.walks, st.emitted, st.emitted_raw, st.kernel_ms, flush=True)
