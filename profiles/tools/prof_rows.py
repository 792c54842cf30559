import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', '..'))
import numpy as np, torch
import paper_1609_04104_b200 as tt
from bench import CONFIGS, make_data, init_factors
cfg = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
T = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg["T"] = T
cl = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ids = list(range(cfg["slices"]))
ks, _ = make_data(cfg, ids)
A0, B0 = init_factors(cfg, ids)
if "vd" in cfg:  # static variable-density rows, as bench.py draws them
    Smax = int(np.ceil(cfg["vd"] * cfg["n"]))
    tab = np.zeros((T, len(ids), Smax), np.int64)
    for si in range(len(ids)):
        gen = np.random.Generator(np.random.Philox(key=2024 + (si << 64)))
        for f in range(T):
            tab[f, si] = tt.variable_density_rows(cfg["n"], -1.0, cfg["vd"], gen)
    pol = tt.StaticRows(tab, np.full((T, len(ids)), Smax))
else:
    pol = tt.Informative(k=cfg["K"], forced=cfg["forced"], beta=cfg["beta"], key0=2024)
eng = tt.OnlineEngine(cfg["n"], cfg["n"], cfg["R"], len(ids), cfg["lam"], tt.Fixed(cfg["mu"]), pol, cluster=cl)
eng.set_image_factors(A0, B0)
ah0, bh0 = eng.ah.clone(), eng.bh.clone()
kd = torch.from_numpy(ks).cuda()
out = eng.make_outputs(T)
args = eng.args(kd, T, out, ah_in=ah0, bh_in=bh0, frame0=0, t0=1)
from paper_1609_04104_b200 import _ops as K
for i in range(3):
    eng.philox_pos.zero_()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); K.track_rows(args); e.record(); torch.cuda.synchronize()
    print(f"launch {i}: {s.elapsed_time(e):.3f} ms  {1000*s.elapsed_time(e)/T:.2f} us/frame  cluster {eng.cluster}")
clk = torch.zeros(T, 32, dtype=torch.int64, device='cuda')
args.phase_clock = clk.data_ptr()
eng.philox_pos.zero_(); K.track_rows(args); torch.cuda.synchronize()
c = clk.cpu().numpy().astype(np.int64)
names = {0: "frame start", 26: "a:colnorm", 1: "a-partials", 2: "B1", 24: "s:nrm", 25: "s:usm", 27: "s:sync",
         28: "s:ahnorm", 3: "s:scores", 4: "B2", 29: "b:scan+cdf", 30: "b:draws", 31: "b:union", 20: "b:end", 5: "draw",
         6: "publishAhS", 7: "B3 complete", 16: "h:tile landed", 17: "h:Z (one tile) / W", 18: "h:Ah_S + GA",
         19: "h:W (one tile) / Z", 8: "heavy-rest", 9: "h/ga/yn", 10: "B4", 11: "Gbuild", 12: "solve", 13: "cost/mu",
         21: "u:mark", 22: "u:P", 23: "u:Q", 14: "update", 15: "outputs"}
from paper_1609_04104_b200 import _lib as L
Smax = eng.max_rows
if L.lib().tt_rows_mirror_fits(cfg["n"], cfg["n"], cfg["R"], Smax, eng.cluster):
    print("mirrored kernel (tt_rows2.cu)")
    names = {0: "frame start", 1: "GB bcast + norms", 2: "scores", 3: "draw / rows", 4: "marks + AhS + GA",
             5: "Y landed", 6: "W + Z GEMMs", 7: "h / yn partials", 8: "B1", 9: "Gram", 10: "solve", 11: "cost/mu",
             12: "Z sums + aown", 16: "P GEMM", 13: "Q GEMM", 17: "apply", 14: "GB scatter", 15: "outputs + B2"}
cc = c[5:]
# stamps present in every frame, ordered by their median offset from the frame start (the one-tile and the
# k-tiled heavy phases stamp 16-19 on different sides of B3)
ks = [k for k in range(32) if (cc[:, k] > 0).all()]
off = {k: np.median(cc[:, k] - cc[:, 0]) for k in ks}
ks.sort(key=lambda k: off[k])
print("cycles per phase (median over frames 5.., each row = time since the previous stamp):")
for p_, k in zip(ks, ks[1:]):
    print(f"  {names.get(k, k):22s} {int(np.median(cc[:, k] - cc[:, p_])):7d}")
fr = np.median(np.diff(cc[:, 0]))
print("frame total", fr, "cycles =", fr / 1.965e3, "us at 1965 MHz")
