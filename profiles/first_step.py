"""Why is the first timed step slower? Per-step device times of the GPT-2 S
set under variants: plain, device sleep before the loop, NVML polling thread,
two consecutive loops."""
import os, sys, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_16932_b200 as pe
import pe_synth as syn
shapes = syn.layer_set_shapes("gpt2-small")
xs = [(torch.randn(s, device="cuda") * 0.02).to(torch.bfloat16) for s in shapes]
ys = [torch.empty_like(x) for x in xs]
ctx = pe.Context(0)
ctx.reserve(shapes)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ctx.polar(xs, ys)
torch.cuda.synchronize()


def loop(tag, sleep=False, flush_on=True, steps=8):
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if sleep:
        torch.cuda._sleep(4_000_000)
    for k in range(steps):
        if flush_on:
            flush.zero_()
        evs[k][0].record()
        ctx.polar(xs, ys)
        evs[k][1].record()
    torch.cuda.synchronize()
    print(tag, [round(a.elapsed_time(b), 3) for a, b in evs], flush=True)


loop("plain")
loop("plain again")
loop("sleep", sleep=True)
loop("noflush", flush_on=False)
loop("noflush sleep", sleep=True, flush_on=False)
stop = [False]
def poll():
    import pynvml
    pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop[0]:
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM); time.sleep(0.002)
t = threading.Thread(target=poll, daemon=True); t.start()
loop("nvml sleep", sleep=True)
stop[0] = True
torch.cuda.synchronize()
time.sleep(0.05)
loop("after 50 ms idle, sleep", sleep=True)
