"""MLEM ms per iteration (K-iteration graph replays, CUDA events), repeated: prints min/median/max."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctis_synth as syn  # noqa: E402
import paper_2006_01573_b200 as ctis  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
solver = sys.argv[3] if len(sys.argv) > 3 else "mlem"   # mlem | monitored | smart
cfg = syn.config(name)
plan = ctis.Plan.from_geometry(cfg.geom, syn.paper_taps(cfg))
plan.set_option(ctis.OPT_VALIDATE_DATA, 0)
if os.environ.get("CTIS_FUSED") is not None:
    plan.set_option(ctis.OPT_FUSED_RATIO, int(os.environ["CTIS_FUSED"]))
g = plan.forward(torch.from_numpy(syn.scene_blobs(cfg.geom).reshape(-1)).cuda())
f = torch.ones(cfg.geom.m, device="cuda")
def run():
    if solver == "monitored":
        plan.mlem_monitored(g, f, K, -1.0)   # never stops early: K iterations with the likelihood trace
    elif solver == "smart":
        plan.smart(g, f, K)
    else:
        plan.mlem(g, f, K)


for _ in range(3):
    run()
ts = []
for _ in range(15):
    f.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3 / K)
ts.sort()
print(f"{name} {solver} pdl={os.environ.get('CTIS_PDL', '0')} fused={os.environ.get('CTIS_FUSED', '1')} launches={plan.last_launch_count()} us/iter min {ts[0]:.1f} med {ts[len(ts) // 2]:.1f} max {ts[-1]:.1f}")
