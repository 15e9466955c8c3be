"""Small workload for compute-sanitizer: every family once through hmdp_compute (FP32 and
FP64; direct path, graph capture, replay), a few device MD steps, a device-DD evaluation,
hybrid device MD (classical force field + DP group)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

s = P.generate_synthetic_system(64)
models = [P.make_model(P.ModelFamily.embed_fit, 1, 0.6, 2, 8, 32, 1),
          P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1),
          P.make_dp_model(P.ModelFamily.se_a, 1), P.make_dp_model(P.ModelFamily.repformer, 2),
          P.make_dp_model(P.ModelFamily.repflow, 2)]
for m in models:
    ctx = P.Context(m, max_atoms=64)
    for prec in (P.Precision.fp32, P.Precision.fp64):
        for _ in range(3):  # direct path, capture, replay
            out = ctx.compute(s.positions, s.types, s.box, prec)
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, 0.001,
                  P.Precision.fp32, steps_per_graph=2)
    md.run(4)
    print(m.family, out.energy, md.state()[3], flush=True)
from paper_2602_02234_b200.dd import DeviceDD, run_local  # noqa: E402

m = models[1]
engs = [DeviceDD(P.Context(m, max_atoms=64), 64, s.types, s.box, (2, 1, 1), r,
                 P.Precision.fp64) for r in range(2)]
for e in engs:
    e.load(s.positions)
run_local(engs)
print("dd", engs[0].result()[0])

# classical force field + hybrid device MD (DP on the protein group)
import oracle as O  # noqa: E402  (topology fixture only)
from paper_2602_02234_b200.ff import ClassicalFF, HybridMD  # noqa: E402
from paper_2602_02234_b200.hybrid import plan_group_preprocessing, synthetic_topology  # noqa: E402

n = 582
sh = P.generate_synthetic_system(n, temperature=300.0)
t = O.ref_synthetic_topology(n)
topo2, plan = plan_group_preprocessing(synthetic_topology(n), "protein")
eo = np.zeros(n + 1, dtype=np.int32)
ex = []
for i in range(n):
    ex += topo2.exclusions[i]
    eo[i + 1] = len(ex)
kept = set(map(tuple, topo2.bonds))
kb = [k for k, b in enumerate(map(tuple, t["bonds"])) if b in kept]
ff = ClassicalFF(sh.types, t["charges"], O.LJ_SIGMA, O.LJ_EPS, eo, np.array(ex), t["bonds"][kb],
                 t["bond_params"][kb], coulomb_scheme=1)
hm = HybridMD(P.Context(models[1], max_atoms=n), ff, plan.atoms, sh.positions, sh.velocities,
              sh.masses, sh.types, sh.box, dt_ps=0.001, precision=P.Precision.fp32,
              steps_per_graph=2)
hm.run(4)
print("hybrid", hm.state()[3])

# round 2: the pull-form message backward at paper size (4114 atoms: 2-warp teams,
# the 28-warp-CTA build, stored z rows) and beyond the z-row budget (32 912 atoms:
# 1-warp teams, z recomputed); the halo-exchange and gather-to-root DD engines
big = P.generate_synthetic_system(4114)
ctxb = P.Context(models[1], max_atoms=4114)
for _ in range(3):  # direct path, capture, replay
    ob = ctxb.compute(big.positions, big.types, big.box, P.Precision.fp32)
print("2PTC", ob.energy, flush=True)
rep = P.replicate(big, (2, 2, 2))
orp = P.Context(models[1], max_atoms=rep.n_atoms).compute(rep.positions, rep.types, rep.box,
                                                          P.Precision.fp32)
print("2PTC x8", orp.energy, flush=True)
from paper_2602_02234_b200 import dd  # noqa: E402

for strategy in ("halo", "gather"):
    hub = dd.Hub(2)
    he = [dd.HaloDD(P.Context(models[1], max_atoms=582), 582, sh.types, sh.box, (2, 1, 1), r,
                    P.Precision.fp32, masses=sh.masses, strategy=strategy) for r in range(2)]
    for e in he:
        e.attach_hub(hub.handle)
        e.load(sh.positions, sh.velocities)
    dd.run_hub(he, "eval")
    dd.run_hub(he, "open", 0.001)
    dd.run_hub(he, "md", 0.001, steps=2)
    print(strategy, he[0].energy_virial()[0], flush=True)
    hub.close()
