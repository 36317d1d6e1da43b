"""Per-launch %globaltimer timeline of the last Gram / poly / update launch
of one pe_polar call, and the clock64 steps of the last tile's epilogue
(PE_DEBUG_GEMM=128; timing experiments on a debug build only:
PE_NVCC_FLAGS=-DPE_GEMM_TIMELINE=1 python -c "import paper_2505_16932_b200.build
as b; b.build(force=True)").  Usage: PE_DEBUG_GEMM=128 python
profiles/phase_timeline.py <rows> <cols> [count] | <workload>."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_16932_b200 as pe  # noqa: E402
import pe_synth as syn  # noqa: E402

if sys.argv[1].isdigit():
    shapes = [(int(sys.argv[1]), int(sys.argv[2]))] * (int(sys.argv[3]) if len(sys.argv) > 3 else 1)
    name = f"{sys.argv[1]}x{sys.argv[2]}x{len(shapes)}"
else:
    shapes = syn.layer_set_shapes(sys.argv[1])
    name = sys.argv[1]
xs = [(torch.randn((r, c), device="cuda") * 0.02).to(torch.bfloat16) for r, c in shapes]
ys = [torch.empty_like(x) for x in xs]
ctx = pe.Context(0)
for _ in range(3):
    ctx.polar(xs, ys, iters=5)
torch.cuda.synchronize()
L = pe.lib()
buf = (ctypes.c_longlong * (8 * 1024))()
assert L.pe_debug_stats(ctx._h, buf) == 0
a = np.array(buf[:6144], dtype=np.int64).reshape(3, 256, 8)[:, :148, :]
ok = a[:, :, 0] > 0
newest = a[:, :, 6].max()
ok &= a[:, :, 0] > newest - 10**9          # this call's launches only (CTAs of a smaller grid never ran)
t0 = a[0, :, 0][ok[0]].min()
labels = ["entry", "pdl done", "1st stage", "last commit", "last store", "stores done", "exit", "last tfull"]
print(f"# {name}: last launch per mode of the 3rd call, us relative to the Gram's first CTA entry")
for mode, nm in enumerate(["gram", "poly", "update"]):
    ent, ext = a[mode, ok[mode], 0], a[mode, ok[mode], 6]
    lo, hi = ent.min(), ext.max()
    cells = []
    for k in (0, 1, 2, 3, 7, 4, 5, 6):
        v = a[mode, ok[mode], k]
        v = v[(v >= lo) & (v <= hi)]
        cells.append(f"{labels[k]} {(v.min() - t0) / 1e3:7.2f}..{(v.max() - t0) / 1e3:7.2f}" if v.size else f"{labels[k]} -")
    print(f"{nm:6s} " + " | ".join(cells))
ep = np.array(buf[:], dtype=np.int64)[6144:6144 + 3 * 512].reshape(3, 64, 8)
elab = ["acc ready", "1st TMEM ld", "1st half", "c0 computed", "c0 store issued", "c1 slot free", "c1 computed", "stores left smem"]
print("# last tile's epilogue, warp 2 of CTAs 0..63: SM cycles after its accumulator is ready (median / max)")
for mode, nm in enumerate(["gram", "poly", "update"]):
    good = ok[mode, :64] & (ep[mode, :, 0] > 0) & (ep[mode, :, 7] >= ep[mode, :, 0])
    if not good.any():
        print(f"{nm:6s} -")
        continue
    cells = []
    for k in range(1, 8):
        d = ep[mode, good, k] - ep[mode, good, 0]
        cells.append(f"{elab[k]} {int(np.median(d))} ({int(d.max())})")
    print(f"{nm:6s} " + " | ".join(cells))
