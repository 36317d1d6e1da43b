"""Tail hiding probe: the GPT-2 S set split into two interleaved halves run
concurrently by two contexts on two streams, vs one call on one stream.
Device time from a common start event to both streams' end."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
import pe_synth as syn
shapes = syn.layer_set_shapes(sys.argv[1] if len(sys.argv) > 1 else "gpt2-small")
xs = [(torch.randn(s, device="cuda") * 0.02).to(torch.bfloat16) for s in shapes]
ys = [torch.empty_like(x) for x in xs]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
c0, c1, c2 = pe.Context(0), pe.Context(0), pe.Context(0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()
for split in ("one", "alt", "half"):
    if split == "alt":
        g1, g2 = list(range(0, len(xs), 2)), list(range(1, len(xs), 2))
    else:
        g1, g2 = list(range(len(xs) // 2)), list(range(len(xs) // 2, len(xs)))
    ts = []
    for rep in range(12):
        flush.zero_()
        if split == "one":
            c0.polar(xs, ys)                       # pre-roll
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            c0.polar(xs, ys)
            b.record()
        else:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2_000_000)
            a.record()
            s1.wait_stream(main)
            s2.wait_stream(main)
            with torch.cuda.stream(s1):
                c1.polar([xs[i] for i in g1], [ys[i] for i in g1])
            with torch.cuda.stream(s2):
                c2.polar([xs[i] for i in g2], [ys[i] for i in g2])
            main.wait_stream(s1)
            main.wait_stream(s2)
            b.record()
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{split}: median {ts[len(ts) // 2]:.4f} ms  min {ts[0]:.4f}", flush=True)
