"""Same-box library context: cuBLAS (torch.matmul) bf16 throughput on the GEMM
shapes of the Polar Express phases, and Listing 2 run eagerly in
PyTorch on the same layer sets.  Context only -- not part of the product path.
Usage: python profiles/cublas_ref.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import pe_synth as syn  # noqa: E402


def bench(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


out = {}
for (M, N, K) in [(8192, 8192, 8192), (4096, 14336, 4096), (4096, 4096, 14336), (4096, 4096, 4096),
                  (768, 3072, 768), (768, 768, 3072), (768, 768, 768)]:
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    y = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    ms = bench(lambda: x @ y)
    out[f"{M}x{N}x{K}"] = round(2 * M * N * K / ms / 1e9, 1)

coeffs = [(8.28721201814563, -23.595886519098837, 17.300387312530933),
          (4.107059111542203, -2.9478499167379106, 0.5448431082926601),
          (3.9486908534822946, -2.908902115962949, 0.5518191394370137),
          (3.3184196573706015, -2.488488024314874, 0.51004894012372),
          (2.300652019954817, -1.6689039845747493, 0.4188073119525673)]
coeffs = [(a / 1.01, b / 1.01 ** 3, c / 1.01 ** 5) for (a, b, c) in coeffs]


def listing2(G):
    X = G.bfloat16()
    tr = G.size(-2) > G.size(-1)
    if tr:
        X = X.mT
    X = X / (X.norm(dim=(-2, -1), keepdim=True) * 1.01 + 1e-7)
    for a, b, c in coeffs:
        A = X @ X.mT
        B = b * A + c * A @ A
        X = a * X + B @ X
    if tr:
        X = X.mT
    return X


compiled = torch.compile(listing2)       # as the paper runs it (@torch.compile)


def batched_by_shape(xs, fn):
    """The strongest plain-PyTorch arrangement: same-shape matrices stacked and
    run as one batched Listing 2 (bmm), one call per shape."""
    groups = {}
    for x in xs:
        groups.setdefault(tuple(x.shape), []).append(x)
    return [fn(torch.stack(g)) for g in groups.values()]


def listing2_batched(G):
    X = G.bfloat16()
    tr = G.size(-2) > G.size(-1)
    if tr:
        X = X.mT
    X = X / (X.norm(dim=(-2, -1), keepdim=True) * 1.01 + 1e-7)
    for a, b, c in coeffs:
        A = X @ X.mT
        B = b * A + c * A @ A
        X = a * X + B @ X
    if tr:
        X = X.mT
    return X


compiled_batched = torch.compile(listing2_batched)
for wl in ("gpt2-small", "llama3-8b"):
    shapes = syn.layer_set_shapes(wl)
    xs = [(torch.randn(r, c, device="cuda") * 0.02).to(torch.bfloat16) for r, c in shapes]
    it = 3 if wl.startswith("llama") else 10
    out[f"listing2_eager_{wl}_ms"] = round(bench(lambda: [listing2(x) for x in xs], iters=it, warm=2), 3)
    out[f"listing2_compiled_{wl}_ms"] = round(bench(lambda: [compiled(x) for x in xs], iters=it, warm=2), 3)
    out[f"listing2_batched_compiled_{wl}_ms"] = round(
        bench(lambda: batched_by_shape(xs, compiled_batched), iters=it, warm=2), 3)
    del xs
    torch.cuda.empty_cache()
print(json.dumps({"cublas_bf16_tflops_and_listing2_ms": out}))
