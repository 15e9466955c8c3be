"""Stage cycle breakdown of k_msg_fwd (dev aid; needs a -DHMDP_TPROBE build at argv[1])."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200._lib as L
L.LIB_PATH = os.path.abspath(sys.argv[1])
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD
lib = L.lib()
name = sys.argv[2] if len(sys.argv) > 2 else "1YRF"
m = P.make_model(P.ModelFamily(1), 3, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(P.PAPER_SYSTEMS[name])
ctx = P.Context(m, max_atoms=s.n_atoms)
md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, steps_per_graph=10)
md.run(20)
buf = (ctypes.c_ulonglong * 32)()
lib.hmdp_debug_tprobe(buf, 1)
K = 100
md.run(K)
lib.hmdp_debug_tprobe(buf, 1)
nwarps = 4 * s.n_atoms  # G=4 teams at 1YRF; per-warp average below
labels = ["stage wait", "pdl_wait", "prologue loads", "edge loop", "team sum", "matvecs fwd", "P push", "fit", "bwd"]
for k, lab in enumerate(labels):
    print(f"{k} {lab:16s} {buf[k] / (K * 2 * nwarps):10.0f} cycles/warp/launch (summed over both msg_fwd kernels)")
