"""Per-step time of the halo-exchange DD program on ONE rank (no peers: the DD
compute path alone -- roles, search of owned+halo rows, push-form network over the
owned list, force, integration) vs the single-domain device MD step, same box."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2602_02234_b200 as P
from paper_2602_02234_b200 import dd
from paper_2602_02234_b200.md import DeviceMD

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4114
m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(n)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
eng = dd.HaloDD(P.Context(m, max_atoms=n), n, s.types, s.box, (1, 1, 1), 0, P.Precision.fp32,
                masses=s.masses, stream=st)
eng.load(s.positions, s.velocities)
eng.step("eval"); eng.step("open", 0.001)
for _ in range(20): eng.step("md", 0.001)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    eng.step("md", 0.001)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 500
e0.record(st)
for _ in range(K): g.replay()
e1.record(st); torch.cuda.synchronize()
dd_us = e0.elapsed_time(e1) / K * 1e3
md = DeviceMD(P.Context(m, max_atoms=n), s.positions, s.velocities, s.masses, s.types, s.box, steps_per_graph=100)
md.run(200); md.state()
t0 = time.perf_counter(); md.run(K); md.state(); sd_us = (time.perf_counter() - t0) / K * 1e6
print(f"n={n}: DD program on one rank {dd_us:.1f} us/step ({eng.launches()} launches so far), single-domain {sd_us:.1f} us/step")
