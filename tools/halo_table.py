"""Halo geometry of the halo-exchange DD on the paper boxes:
owned / halo atoms and halo bytes per rank for one box split over 2x1x1, 2x2x1, 2x2x2,
measured by the engine itself (ranks simulated as contexts on one GPU, in-process hub),
plus an FP64 single-domain check of every configuration.
usage: python tools/halo_table.py > profiles/round2/halo_table.md"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200 import dd

E1 = {"1YRF": {2: (298, 297), 4: (154, 396), 8: (94, 402)},
      "1UBQ": {2: (616, 439), 4: (324, 580), 8: (171, 539)},
      "3LZM": {2: (1323, 756), 4: (686, 922), 8: (343, 842)},
      "2PTC": {2: (2060, 1049), 4: (1052, 1240), 8: (620, 1066)}}

print("# Halo-exchange DD: owned / halo atoms per rank vs SURVEY table E1\n")
print("Measured by `HaloDD.roles()` after one evaluation (ranks simulated on one B200 through "
      "the in-process hub, the same C++ step program the NCCL transport runs); halo bytes = "
      "useful rows x row bytes over every round of one DPA3 MD step in FP64 (P rows 256 B; FP32 halves them) (POS x+v, P^l and "
      "dE/dh sums per layer, forces, (E, W)); E = the decomposed energy vs the single-domain "
      "one (FP64).\n")
print("| box | ranks | max owned (E1) | max halo (E1) | rank-0 halo bytes / step | "
      "transferred (fixed-capacity packets) | dE/E vs single domain |")
print("|---|---|---|---|---|---|---|")
m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
for system, n in P.PAPER_SYSTEMS.items():
    s = P.generate_synthetic_system(n, temperature=300.0)
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64).energy
    for world in (2, 4, 8):
        dims = dd.rank_grid(world)
        hub = dd.Hub(world)
        engs = [dd.HaloDD(P.Context(m, max_atoms=n), n, s.types, s.box, dims, r,
                          P.Precision.fp64, masses=s.masses) for r in range(world)]
        for e in engs:
            e.attach_hub(hub.handle)
            e.load(s.positions, s.velocities)
        dd.run_hub(engs, "eval")
        roles = [e.roles() for e in engs]
        own = max(int((r == 1).sum()) for r in roles)
        halo = max(int((r == 2).sum()) for r in roles)
        st = engs[0].halo_stats()
        E = engs[0].energy_virial()[0]
        eo, eh = E1[system][world]
        print(f"| {system} | {world} ({dims[0]}x{dims[1]}x{dims[2]}) | {own} ({eo}) | {halo} ({eh}) | "
              f"{st['halo_bytes_per_step'] / 1e3:.0f} KB | "
              f"{st['transferred_bytes_per_step'] / 1e3:.0f} KB | {abs(E - ref) / abs(ref):.1e} |",
              flush=True)
        for e in engs:
            e.ctx.close()
        hub.close()
