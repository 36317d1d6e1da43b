#!/usr/bin/env python
"""Benchmark of the Polar Express hot path on B200 (BASELINE.json metric:
"polar factors/s and TFLOP/s (fraction of bf16 tensor peak) at 1/2/4/8 B200").

One step = one pe_polar call over a whole Muon layer set (all §8(a) rows:
Frobenius norm, scale/orient, T x {Gram, b A + c A^2, a X + B X}, transpose
back), inputs resident in HBM.  Default workload: the north-star
configuration (BASELINE.json north_star / configs[3]): the full Llama-3-8B
Muon layer set, 224 matrices, bf16, T=5, degree 5 (reading R12); the GPT-2
Small / Large sets (configs[1], [2]) are reported under `extra_workloads`.  With N ranks each
rank computes its pe_shard_plan share and the results are all-gathered
over NCCL inside libpe (pe_polar_sharded; strong scaling of one layer set).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                       [--impl ours|reference] [--extra gpt2-small,...]
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "polar factors/s and TFLOP/s (fraction of bf16 tensor peak) at 1/2/4/8 B200"
UNIT = "matrices/s"
STD = 0.02          # momentum-like N(0, 0.02^2) entries (scale-invariant method)
ELL, DEGREE = 1e-3, 5

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """Clocks and throttle reasons DURING the timed region (B200_PROFILING.md
    clocks line): NVML polled every ~2 ms from a thread while `active` (the
    timed steps, host enqueue to device completion); nvidia-smi at 200 ms if
    NVML is unavailable."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []
        self.nvml = None
        self.samples = []          # (sm_mhz, max_mhz, reasons bitmask)
        self.active = False
        self._stop = False

    def start(self):
        if os.environ.get("PE_BENCH_SAMPLER") == "smi":     # A/B knob: skip NVML
            self.nvml = None
            return self._start_smi()
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            try:
                pr = torch.cuda.get_device_properties(self.device)
                h = pynvml.nvmlDeviceGetHandleByPciBusId(
                    f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.nvml, self.h = pynvml, h
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        self._start_smi()

    def _start_smi(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        while not self._stop:
            if self.active:
                try:
                    sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.samples.append((float(sm), float(mx), int(rs)))
                except Exception:
                    pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            if self.active:
                self.lines.append(line.strip())

    def stop(self):
        self._stop = True
        if self.nvml is None and not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no NVML / nvidia-smi"]}
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        if self.nvml is not None:
            rows = self.samples
            src = "nvml 2 ms, timed steps only"
        else:
            rows = []
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                try:
                    bits = int(parts[3], 16) if parts[3].startswith("0x") else int(parts[3])
                    rows.append((float(parts[0]), float(parts[1]), bits))
                except (ValueError, IndexError):
                    continue
            src = "nvidia-smi 200 ms, timed steps only"
        for a, b, bits in rows:
            sm.append(a)
            smax.append(b)
            for bit, name in REASON_BITS.items():
                if bits & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "sampler": src}


def layer_set(name):
    import pe_synth as syn
    return syn.layer_set_shapes(name.split(":")[0])


def rect_restart(name):
    """'<set>:alg4r<k>' runs the set with App. H's Alg. 4 (pe_set_rect_iteration,
    restart every k iterations, shift 1e-3) on the matrices past the aspect
    rule alpha > 1.5 T / (T - 1); 0 = Listing 2."""
    tag = name.split(":")[1] if ":" in name else ""
    return int(tag[len("alg4r"):]) if tag.startswith("alg4r") else 0


def alg4_flops(shapes, T, restart):
    """Algorithmic flops of a call with Alg. 4 on the qualifying matrices
    (symmetric products counted once): per application
    3 l s^2 (Y, X Q) + s^3 (h_1's square) + 6 s^3 per further iteration
    (Y Q, Q^T (Y Q) upper half, R^2, H Q); the others pe_flops' count."""
    thr = 1.5 * T / (T - 1) if T > 1 else float("inf")
    f = 0.0
    for r, c in shapes:
        s_, l_ = min(r, c), max(r, c)
        if restart > 0 and s_ > 128 and l_ > thr * s_:
            k = min(restart, T)
            for t0 in range(0, T, k):
                kb = min(k, T - t0)
                f += 3.0 * l_ * s_ * s_ + s_ ** 3 + 6.0 * (kb - 1) * s_ ** 3
        else:
            f += T * (s_ * (s_ + 1) * l_ + s_ * s_ * (s_ + 1) + 2.0 * s_ * s_ * l_)
    return f


def make_inputs(shapes, idx, device, seed=0):
    import torch
    g = torch.Generator(device=device)
    xs = []
    for i in idx:
        g.manual_seed(seed * 100003 + i)
        r, c = shapes[i]
        xs.append((torch.randn((r, c), generator=g, device=device, dtype=torch.float32) * STD).to(torch.bfloat16))
    return xs


def kind_work(shapes, T):
    """Algorithmic work per launch of each kernel kind."""
    fl = {"gram": 0.0, "poly": 0.0, "update": 0.0}
    by = {"norm": 0.0, "scale": 0.0, "transpose_back": 0.0}
    for r, c in shapes:
        m, n = min(r, c), max(r, c)
        fl["gram"] += m * (m + 1) * n
        fl["poly"] += m * m * (m + 1)
        fl["update"] += 2.0 * m * m * n
        by["norm"] += 2.0 * m * n
        if c % 8:                       # bf16 rows that are not 16-byte multiples: copy passes
            by["scale"] += 4.0 * m * n
            by["transpose_back"] += 4.0 * m * n
    fl["fused"] = T * (fl["gram"] + fl["poly"] + fl["update"])    # one launch runs all 3T phases
    return fl, by


def roofline(prof, shapes, T, step_ms, peaks, src, workload=None):
    fl, by = kind_work(shapes, T)
    kind = max(prof, key=lambda k: prof[k][0])
    tot, cnt = prof[kind]
    per_launch_ms = tot / max(cnt, 1)
    sustained = step_ms > 50.0
    traffic, traffic_src, ncu_kind = None, None, None
    try:
        # written by profiles/ncu_traffic.py from an `ncu --set full` capture
        # (dram__bytes_read.sum + dram__bytes_write.sum of that kernel)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f).get(workload or "", {})
            traffic, traffic_src = tj.get(kind), tj.get("_source")
            ncu_kind = tj.get(kind + "_ncu")
    except Exception:
        pass
    if kind in fl:
        achieved = fl[kind] / (per_launch_ms * 1e-3) / 1e12
        peak = peaks["bf16_tflops_sustained" if sustained else "bf16_tflops"]
        out = {"bound": "tensor", "unit": "TFLOP/s"}
    else:
        achieved = by[kind] / (per_launch_ms * 1e-3) / 1e9
        peak = peaks["hbm_gbs"]
        out = {"bound": "hbm", "unit": "GB/s"}
    out.update({"kernel": f"pe_gemm_sm100[{kind}]" if kind in fl else kind, "achieved": round(achieved, 2),
                "peak": peak, "peak_source": f"{src} {'sustained' if (sustained and kind in fl) else 'burst'}",
                "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                "ncu": ncu_kind,
                "algorithmic_per_launch": (fl[kind] if kind in fl else by[kind]),
                "launch_ms": round(per_launch_ms, 4),
                "timing": "CUDA events around each launch of this kernel, on its stream, in a second pass of the same K steps",
                "share_of_step": round(tot / max(sum(v[0] for v in prof.values()), 1e-9), 4)})
    return out


def kernel_table(prof, shapes, T, step_ms, peaks):
    """Every launched kernel kind against its own roofline (same event timing
    and algorithmic counts as `roofline`, which reports the dominant one)."""
    fl, by = kind_work(shapes, T)
    sustained = step_ms > 50.0
    out = {}
    for kind, (tot, cnt) in prof.items():
        if cnt <= 0 or tot <= 0 or (kind not in fl and kind not in by):
            continue
        per = tot / cnt
        if kind in fl:
            a = fl[kind] / (per * 1e-3) / 1e12
            pk = peaks["bf16_tflops_sustained" if sustained else "bf16_tflops"]
            out[kind] = {"bound": "tensor", "unit": "TFLOP/s", "achieved": round(a, 2), "peak": pk,
                         "frac": round(a / pk, 4), "launch_ms": round(per, 4), "launches": cnt}
        else:
            a = by[kind] / (per * 1e-3) / 1e9
            pk = peaks["hbm_gbs"]
            out[kind] = {"bound": "hbm", "unit": "GB/s", "achieved": round(a, 1), "peak": pk,
                         "frac": round(a / pk, 4), "launch_ms": round(per, 4), "launches": cnt}
    return out


def pctl(ms):
    """median / p10 / p90 of per-step device times."""
    v = sorted(ms)
    q = lambda f: v[min(len(v) - 1, max(0, int(round(f * (len(v) - 1)))))]
    return {"median_ms": round(q(0.5), 4), "p10_ms": round(q(0.1), 4), "p90_ms": round(q(0.9), 4),
            "mean_ms": round(sum(v) / len(v), 4), "n": len(v), "all_ms": [round(x, 4) for x in ms]}


def norm_gbs(prof, shapes, steps, peaks):
    """Achieved HBM bandwidth of the norm pass (row a3: m*n elements read)."""
    tot, cnt = prof.get("norm", (0.0, 0))
    if cnt == 0 or tot <= 0:
        return None
    nbytes = sum(2.0 * r * c for r, c in shapes)
    gbs = nbytes / (tot / cnt * 1e-3) / 1e9
    return {"bytes_per_launch": nbytes, "launch_ms": round(tot / cnt, 4), "achieved_gbs": round(gbs, 1),
            "peak_gbs": peaks["hbm_gbs"], "frac": round(gbs / peaks["hbm_gbs"], 4)}


def oracle_time(shapes, T, budget_s=10.0, max_s=30.0, seed=0, steps=None):
    """The fp64 oracle (as it stands) on host cores over a bounded sample.
    steps=None: repeat the sample for ~budget_s; steps=K: exactly K passes
    (the reference arm's timed steps, one pass each)."""
    import pe_synth as syn
    from oracle import coeffs as oc, iteration as oi
    table, _ = oc.pe_coeffs(ELL, DEGREE, 8, 1.01)
    # sample: the first layer's matrices (or the first matrix for big sets)
    nl = {"gpt2-small": 12, "gpt2-small-fused": 12, "gpt2-large": 36}.get(_workload_name[0], 32)
    per_layer = max(1, len(shapes) // nl)
    sample = list(range(per_layer))
    if sum(min(shapes[i]) ** 2 * max(shapes[i]) for i in sample) > 4e11:
        sample = [min(range(len(shapes)), key=lambda i: min(shapes[i]) ** 2 * max(shapes[i]))]
    mats = [syn.gaussian(*shapes[i], seed=seed + i, std=STD) for i in sample]
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        cores = max((d.get("num_threads", 0) for d in info), default=os.cpu_count())
        blas = ",".join(sorted({d.get("internal_api", "?") for d in info}))
    except Exception:
        cores, blas = os.cpu_count(), "?"
    passes, t0 = 0, time.perf_counter()
    step_s = []
    while True:
        ts = time.perf_counter()
        for M in mats:
            oi.polar_express(M, table, T)
        step_s.append(time.perf_counter() - ts)
        passes += 1
        el = time.perf_counter() - t0
        if steps is not None:
            if passes >= steps:
                break
        elif el >= budget_s or el * (passes + 1) / passes > max_s:
            break
    dense = lambda s: T * (4 * min(s) ** 2 * max(s) + 2 * min(s) ** 3)
    f_sample = sum(dense(shapes[i]) for i in sample)
    f_set = sum(dense(s) for s in shapes)
    t_sample = el / passes
    t_set = t_sample * f_set / f_sample
    return {"value": round(len(shapes) / t_set, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{len(sample)} of {len(shapes)} matrices ({'x'.join(map(str, shapes[sample[0]]))}"
                      f"{' ...' if len(sample) > 1 else ''}), {passes} passes in {el:.1f}s, "
                      f"numpy fp64 ({blas}); value = set size / set time extrapolated by the dense-flop ratio "
                      f"{f_set / f_sample:.1f}",
            "sample_ms_per_pass": round(1e3 * t_sample, 3), "step_ms": [round(1e3 * x, 3) for x in step_s],
            "s_per_set_extrapolated": round(t_set, 3), "gflops_fp64": round(f_sample / t_sample / 1e9, 2)}


_workload_name = ["llama3-8b"]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    shapes = layer_set(args.workload)
    # each step = one pass of the oracle over the bounded sample (timed; the
    # warm-up passes are run and discarded); `value` extrapolates the sample's
    # rate to the whole set by the dense-flop ratio, `ms_per_step` is what one
    # timed step took
    oracle_time(shapes, args.iters, steps=max(0, args.warmup)) if args.warmup > 0 else None
    cb = oracle_time(shapes, args.iters, steps=max(1, args.steps))
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cb["sample_ms_per_pass"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "matrices": len(shapes), "T": args.iters, "degree": DEGREE,
                       "ell": ELL},
            "note": "reference = the fp64 CPU oracle (the tier has no reference implementation); one step = one "
                    "pass over the sample named in cpu_baseline.sample, ms_per_step its measured time; value "
                    "extrapolates to the whole set (s_per_set_extrapolated)",
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def time_workload(ctx, shapes, T, steps, warmup, world, rank, device, flush, dist_on, clocks=None, rect=0):
    """Device-timed steps of one layer set; returns per-step ms list, profile, extras."""
    import torch
    import paper_2505_16932_b200 as pe  # noqa: F401
    from paper_2505_16932_b200 import dist as pdist
    idx, owner = pdist.owned(shapes, rank, world) if world > 1 else (list(range(len(shapes))), [0] * len(shapes))
    xs = make_inputs(shapes, idx, device)
    if dist_on and world > 1:
        # pe_polar_sharded: this rank computes its pe_shard_plan share; libpe
        # broadcasts every result from its owner into every rank's output
        # over its own NCCL communicator, bucket by bucket, overlapping compute
        pdist.attach(ctx)
        xin = [None] * len(shapes)
        for i, x in zip(idx, xs):
            xin[i] = x
        # outputs in the pe_shard_layout buffer: each rank's last update
        # epilogues write its chunk, one in-place all-gather per bucket
        _flat, ys = pdist.sharded_outputs(shapes, world, torch.bfloat16, device)
    else:
        ys = [torch.empty_like(x) for x in xs]
    ctx.reserve([shapes[i] for i in idx])
    if rect:
        ctx.set_rect_iteration(rect, 0.0, 1e-3)
    stream = torch.cuda.current_stream(device)

    def step():
        if dist_on and world > 1:
            ctx.polar_sharded(xin, ys, iters=T, stream=stream)
        else:
            ctx.polar(xs, ys, iters=T, stream=stream)

    for _ in range(max(0, warmup - 1)):        # + 1 inside timed(), right before the timed steps
        flush.zero_()                          # warm-up steps see the same flushed L2 as timed ones
        step()
    torch.cuda.synchronize(device)
    launches = ctx.last_launch_count()

    def timed(profile):
        if dist_on:
            torch.distributed.barrier()
        torch.cuda.synchronize(device)
        if clocks is not None and not profile:
            clocks.active = True
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        # the last warm-up step is enqueued right before the timed ones (no
        # idle gap before the first timed step).  Warm-up steps flush L2 like
        # the timed ones: the first write to the 256 MiB flush buffer made the
        # following step ~0.2 ms slower (profiles/first_step.py), which used to
        # land on timed step 1.
        flush.zero_()
        step()
        ctx.profile_enable(profile)          # the K timed steps only (not the warm-up step above)
        for k in range(steps):
            flush.zero_()                    # evict L2 (buffer > 126 MB) between timed steps
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize(device)
        if clocks is not None:
            clocks.active = False
        if dist_on:
            torch.distributed.barrier()
        prof = ctx.profile_read() if profile else None
        ctx.profile_enable(False)
        return [a.elapsed_time(b) for a, b in evs], prof

    # headline: no per-launch events inside the step (they would break the
    # programmatic-dependent-launch overlap between kernels); a second pass
    # with per-launch events gives the per-kernel split and the roofline
    ms, _ = timed(False)
    _, prof = timed(True)
    graph_ms = None
    if not (dist_on and world > 1) and not rect:
        # the whole layer set replayed from one CUDA graph (the
        # reserved plan: no allocation or synchronisation while capturing)
        try:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=torch.cuda.Stream(device)):
                ctx.polar(xs, ys, iters=T, stream=torch.cuda.current_stream(device))
            gr.replay()
            torch.cuda.synchronize(device)
            gevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for k in range(steps):
                flush.zero_()
                gevs[k][0].record()
                gr.replay()
                gevs[k][1].record()
            torch.cuda.synchronize(device)
            graph_ms = [a.elapsed_time(b) for a, b in gevs]
            del gr
        except Exception as e:                       # reported, not fatal
            graph_ms = str(e)[:200]
    if dist_on and world > 1:
        # SURVEY §8(d) multi-GPU: the compute span (this rank's pe_polar on its
        # share) and the exchange span in isolation (pe_sharded_exchange: the
        # library's own per-bucket all-gathers on the same buffers), next to
        # the overlapped pe_polar_sharded step above
        ys_own = [ys[i] for i in idx]

        def span(fn, reps=max(3, steps)):
            out = []
            for _ in range(reps):
                torch.distributed.barrier()
                torch.cuda.synchronize(device)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize(device)
                out.append(a.elapsed_time(b))
            t = torch.tensor([sorted(out)[len(out) // 2]], device=device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            return round(float(t.item()), 4)

        def exchange():
            ctx.sharded_exchange(ys, stream=stream)

        try:
            graph_ms = {"compute_ms": span(lambda: ctx.polar(xs, ys_own, iters=T, stream=stream)),
                        "exchange_ms": span(exchange),
                        "buckets": pe.pe_shard_nbuckets(shapes, world),
                        "note": "max over ranks of the median; exchange = pe_sharded_exchange (libpe's per-bucket "
                                "in-place NCCL all-gathers over the pe_shard_layout buffer); the timed step "
                                "overlaps compute and exchange"}
        except Exception as e:                       # reported, never fatal
            graph_ms = {"error": str(e)[:200]}
    return ms, prof, launches, idx, xs, ys, graph_ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="llama3-8b")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--extra", default="gpt2-small,gpt2-large,llama3-8b-literal,llama3-8b:alg4r3,gpt2-large:alg4r3,gpt2-small:alg4r3",
                    help="comma list of extra layer sets (N=1 only; '<set>:alg4r<k>' = with App. H Alg. 4), or ''")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    _workload_name[0] = args.workload
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import paper_2505_16932_b200 as pe

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    dist_on = world > 1
    if dist_on:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    ctx = pe.Context(local_rank)
    peaks, src = measured_peaks()
    T = args.iters
    shapes = layer_set(args.workload)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)

    clocks = ClockSampler(local_rank)
    clocks.start()
    ms, prof, launches, idx, xs, ys, graph_ms = time_workload(ctx, shapes, T, args.steps, args.warmup, world,
                                                              rank, device, flush, dist_on, clocks)
    clk = clocks.stop()
    mean_ms = sum(ms) / len(ms)
    if dist_on:
        t = torch.tensor([mean_ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        mean_ms = float(t.item())
    flops = pe.pe_flops(shapes, T, DEGREE)
    value = len(shapes) / (mean_ms * 1e-3)
    tflops = flops / (mean_ms * 1e-3) / 1e12
    peak_key = "bf16_tflops_sustained" if mean_ms > 50 else "bf16_tflops"

    # e2e through the public API on pinned host buffers (H2D + D2H inside)
    hin = [x.cpu().pin_memory() for x in xs]
    hout = [torch.empty_like(h).pin_memory() for h in hin]
    e2e_ms = []
    if not dist_on:
        ctx.polar_host(hin, hout, iters=T)
        for _ in range(max(3, min(args.steps, 10))):
            t0 = time.perf_counter()
            ctx.polar_host(hin, hout, iters=T)      # synchronises its stream
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_note = ("pe_polar_host on pinned host tensors, wall clock per call (host->device copies, compute, "
                    "device->host copies; synchronises): the batch is pipelined in groups so the PCIe transfers "
                    "(both directions concurrently) hide behind the compute except the first group's H2D and "
                    "the last group's D2H; no L2 flush between calls")
    else:
        # N ranks: each rank's owned inputs in from pinned host memory, the
        # sharded call (compute + libpe's all-gather: every rank ends with every
        # result), its owned results out to pinned host memory (the union over
        # ranks is the whole set); wall clock between barriers, max over ranks
        stream = torch.cuda.current_stream(device)
        xin_e = [None] * len(shapes)
        for i, x in zip(idx, xs):
            xin_e[i] = x
        ys_e = ys
        for k in range(max(3, min(args.steps, 10)) + 1):
            torch.distributed.barrier()
            torch.cuda.synchronize(device)
            t0 = time.perf_counter()
            for x, h in zip(xs, hin):
                x.copy_(h, non_blocking=True)
            ctx.polar_sharded(xin_e, ys_e, iters=T, stream=stream)
            for i, h in zip(idx, hout):
                h.copy_(ys_e[i], non_blocking=True)
            torch.cuda.synchronize(device)
            if k > 0:                                   # the first pass is a warm-up
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_note = ("per rank: its owned inputs host->device from pinned memory, pe_polar_sharded (compute + "
                    "libpe's per-bucket all-gather, every rank ends with every result), its owned results "
                    "device->host into pinned memory; wall clock between barriers, max over ranks")
    e2e_mean = sum(e2e_ms) / len(e2e_ms)
    if dist_on:
        t = torch.tensor([e2e_mean], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_mean = float(t.item())
    io_bytes = sum(x.numel() * 2 for x in xs)

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(mean_ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: seeded N(0, 0.02^2) bf16 momentum matrices generated on device",
        "config": {"workload": args.workload, "matrices": len(shapes), "T": T, "degree": DEGREE, "ell": ELL,
                   "coeffs": "pe_coeffs(1e-3,5,8,1.01) (Listing 2 table)",
                   "l2": "flushed between timed steps (256 MiB write, outside the events)",
                   "parallelism": f"dp{world} (pe_polar_sharded: bucket-balanced LPT shard + per-bucket in-place "
                                  f"NCCL all-gather)" if world > 1 else "single GPU"},
        "tflops": round(tflops, 2), "tflops_unit": "TFLOP/s (algorithmic, symmetric-aware)",
        "tflops_dense": round(sum(T * (4.0 * min(s_) ** 2 * max(s_) + 2.0 * min(s_) ** 3) for s_ in shapes)
                              / (mean_ms * 1e-3) / 1e12, 2),
        "tflops_dense_unit": "TFLOP/s counting every product dense (the paper's MAC model x 2, SURVEY §8d); "
                             "not comparable with `tflops`",
        "frac_of_bf16_peak": round(tflops / peaks[peak_key], 4),
        "frac_of_bf16_peak_sustained": round(tflops / peaks["bf16_tflops_sustained"], 4),
        "layer_sets_per_s": round(1e3 / mean_ms, 3),
        "peak_used": f"{peaks[peak_key]} TFLOP/s ({src} {'sustained' if peak_key.endswith('sustained') else 'burst'})",
        "e2e": {"value": round(len(shapes) / (e2e_mean * 1e-3), 3), "unit": UNIT,
                "ms_per_step": round(e2e_mean, 3),
                "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": io_bytes, "note": e2e_note},
        "gpu_launches": launches * args.steps,
        "clocks": clk,
        "roofline": roofline(prof, [shapes[i] for i in idx], T, mean_ms, peaks, src, args.workload),
        "per_kernel_roofline": kernel_table(prof, [shapes[i] for i in idx], T, mean_ms, peaks),
        "per_kernel_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in prof.items()},
        "ms_per_step_stats": pctl(ms),
        "graph_replay": (pctl(graph_ms) if isinstance(graph_ms, list) else (None if world > 1 else graph_ms)),
        "multi_gpu_spans": graph_ms if world > 1 else None,
        "norm_pass": norm_gbs(prof, [shapes[i] for i in idx], args.steps, peaks),
    }

    # extra layer sets (north-star Llama-3-8B) at N=1
    extras = {}
    if world == 1 and args.extra:
        del xs, ys, hin, hout
        for name in [s for s in args.extra.split(",") if s and s != args.workload]:
            time.sleep(3.0)        # let the power limiter recover after the previous (long) workload
            sh = layer_set(name)
            ctx2 = pe.Context(local_rank)
            c2 = ClockSampler(local_rank)
            c2.start()
            st2 = 10
            rk = rect_restart(name)
            ms2, prof2, l2, idx2, xs2, ys2, _ = time_workload(ctx2, sh, T, st2, 3, 1, 0, device, flush, False, c2,
                                                              rect=rk)
            ck2 = c2.stop()
            m2 = sum(ms2) / len(ms2)
            f2 = alg4_flops(sh, T, rk) if rk else pe.pe_flops(sh, T, DEGREE)
            extras[name] = {"matrices": len(sh), "value": round(len(sh) / (m2 * 1e-3), 3), "unit": UNIT,
                            "ms_per_step": round(m2, 3), "steps": st2, "warmup": 3,
                            "tflops": round(f2 / (m2 * 1e-3) / 1e12, 2),
                            "frac_of_bf16_peak_sustained": round(f2 / (m2 * 1e-3) / 1e12 / peaks["bf16_tflops_sustained"], 4),
                            "frac_of_bf16_peak_burst": round(f2 / (m2 * 1e-3) / 1e12 / peaks["bf16_tflops"], 4),
                            "roofline": None if rk else roofline(prof2, sh, T, m2, peaks, src, name),
                            "per_kernel_roofline": None if rk else kernel_table(prof2, sh, T, m2, peaks),
                            "method": (f"App. H Alg. 4 (restart {rk}, shift 1e-3) on the matrices with aspect "
                                       f"> 1.5 T / (T - 1); tflops from its own algorithmic count" if rk
                                       else "Listing 2"),
                            "per_kernel_ms_per_step": {k: round(v[0] / st2, 4) for k, v in prof2.items()},
                            "clocks": ck2}
            del xs2, ys2
            ctx2.close()
            torch.cuda.empty_cache()
        line["extra_workloads"] = extras

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = oracle_time(shapes, T)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist_on:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
