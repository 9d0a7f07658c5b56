import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2412_06198_b200 import runtime as R
n = 32768
q, k, v = bench.synth_inputs(0, n)
dev = torch.device("cuda")
qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(x)).bfloat16().to(dev) for x in (q, k, v))
plan = R.PrefillPlan(1, 32, 8, n, 128, "auto")
ws = R._workspace(plan.ws_bytes, dev)
out = torch.empty((1, n, 4096), dtype=torch.bfloat16, device=dev)
def step():
    plan.select(qd, kd, ws); plan.run(qd, kd, vd, out, ws)
for _ in range(3): step()
torch.cuda.synchronize()
def t(fn, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
print("eager", t(step))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    step(); torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        step()
torch.cuda.synchronize()
ref = out.clone()
print("graph", t(g.replay))
g.replay(); torch.cuda.synchronize()
print("same output", torch.equal(ref, out))
