#!/usr/bin/env python3
"""Benchmark of the per-block batched execution path (BASELINE.json metric: block-chain decode
tokens/s, per-kernel % of roofline).

One step = one lockstep decode token for every request of the C2 workload (BASELINE.json
configs[1]: Llama-2-7B-shaped synthetic, 32 layers in 4-layer blocks, 4 tenants sharing the first
24 layers, mixed batch 64, prompt 512, decode 128): 6 shared blocks at 64 rows and 8 private
blocks at 16 rows, each a gather -> 4 decoder layers (tcgen05 GEMMs, paged attention) -> scatter,
replayed as one CUDA graph. Inputs (weights 22.7 GB, KV ~21 GB) are far larger than L2.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun each rank serves its own replica of the workload (one GPU each, no data-path
collective: scaling "weak"); rank 0 prints one JSON line.
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

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return dict(PEAKS_FALLBACK), "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML polled every 10 ms on
    a thread (nvidia-smi's own 200 ms loop as the fallback), so even a ~0.25 s region holds
    dozens of samples."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, period_s: float = 0.01):
        self.gpu = gpu
        self.period = period_s
        self.proc = None
        self.nvml = None
        self.samples = []  # (time, sm_mhz, max_mhz, frozenset(reasons))
        self.t = None
        self.t0 = 0.0
        self.stop_ev = threading.Event()

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            self.nvml = (N, h, bits, mx)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        N, h, bits, mx = self.nvml
        while not self.stop_ev.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((time.time(), float(sm), float(mx),
                                     frozenset(n for n, b in bits.items() if r & b)))
            except Exception:
                pass
            self.stop_ev.wait(self.period)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                self.samples.append((time.time(), float(parts[0]), float(parts[1]), frozenset(
                    n for n, v in zip(self.NAMES, parts[3:7]) if v.lower().startswith("active"))))
            except ValueError:
                continue

    def mark(self):
        """Start of the timed region (the sampler runs from before warm-up, so samples exist)."""
        self.t0 = time.time()

    def stop(self):
        if self.nvml is None and self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self.stop_ev.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=1)
        inside = [s for s in self.samples if s[0] >= self.t0]
        if not inside and self.samples:  # region shorter than the sampling period: nearest sample
            inside = [self.samples[-1]]
        reasons = set()
        for s in inside:
            reasons |= s[3]
        return {"sm_mhz": statistics.median(s[1] for s in inside) if inside else None,
                "sm_max_mhz": max(s[2] for s in inside) if inside else None,
                "reasons": sorted(reasons), "samples": len(inside),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------------------------ CPU leg
class CpuDecodeStep:
    """TEST INFRASTRUCTURE (the cpu_baseline leg and --impl reference only): one whole lockstep
    decode step of the workload restated on the host by the oracle (fp32 C, OpenMP over
    `threads`): every block run of the step at its own per-block batch (C2: 6 shared blocks at 64
    rows, 8 private blocks at 16 rows), each row attending over `ctx` tokens of K/V. Blocks with
    the same batch size share one restated weight set (the arithmetic does not depend on the
    values; the host holds ~3.2 GB fp32 per 7B 4-layer block), so memory stays bounded."""

    def __init__(self, wl, threads: int, ctx: int | None = None):
        import numpy as np
        from oracle import oracle as O
        self.wl, self.threads = wl, threads
        self.rows = [r for r in wl.rows_at_block() if r > 0]
        self.ctx = ctx or min(wl.req_prompt[0] + wl.req_output[0] // 2, wl.shape.max_pos - 2)
        self.blocks, self.seqs, self.x = {}, {}, {}
        for r in sorted(set(self.rows)):
            ob = O.OracleBlock(wl.shape, f"cpu-step-{r}", seed=wl.seed)
            seqs = [ob.new_seq(self.ctx + 1) for _ in range(r)]
            for q in seqs:
                q.fill(self.ctx)
            self.blocks[r], self.seqs[r] = ob, seqs
            self.x[r] = np.random.default_rng(r).standard_normal(
                (r, wl.shape.d_model)).astype(np.float32)

    def step(self) -> float:
        """Seconds for one decode step (all block runs, in chain-position order)."""
        t0 = time.perf_counter()
        for r in self.rows:
            self.blocks[r].forward(self.seqs[r], list(range(r)), [self.ctx] * r, self.x[r],
                                   threads=self.threads)
        return time.perf_counter() - t0

    def sample(self) -> str:
        from collections import Counter
        c = Counter(self.rows)
        return ("one whole decode step per sample: " + " + ".join(
            f"{n} block runs at {r} rows" for r, n in sorted(c.items(), reverse=True))
            + f", context {self.ctx}, oracle fp32 C restatement (OpenMP)")


def blocksim_run(wl):
    """TEST INFRASTRUCTURE: the reference's own CPU path - blocksim's Simulation::run (the
    unmodified reference sources in oracle/_ref, scenario.cpp:152-175) on the same requests over
    a zoo of the config's shape (a foundation plus one LoRA variant per tenant from the first
    private layer up, partitioned by the reference), single-threaded as the simulator is. It
    prices block runs from cost tables and computes no tensors. None if oracle/_ref is absent."""
    import json as _j
    import numpy as np
    try:
        from oracle import refshim as R
        if not R.available():
            return None
        L = R.lib()
    except Exception:
        return None
    s = wl.shape
    n_pos = max(len(c) for c in wl.chains)
    shared = set.intersection(*[set(c) for c in wl.chains]) if len(wl.chains) > 1 else set()
    n_shared = sum(1 for b in wl.chains[0] if b in shared)
    p = np.ascontiguousarray(wl.req_prompt, np.int32)
    o = np.ascontiguousarray(wl.req_output, np.int32)
    t0 = time.perf_counter()
    h = L.rs_sim_run(n_pos * s.n_layers, s.d_model, len(wl.chains), n_shared * s.n_layers,
                     wl.n_requests, p.ctypes.data, o.ctypes.data, wl.max_batch_tokens, 0)
    wall = time.perf_counter() - t0
    try:
        err = L.rs_sim_error(h).decode()
        if err:
            return {"error": err}
        rep = _j.loads(L.rs_sim_report(h).decode())
        nb = L.rs_sim_n_batches(h)
    finally:
        L.rs_sim_free(h)
    return {"wall_s": round(wall, 4), "cores": 1, "kind": "reference",
            "what": "blocksim Simulation::run (oracle/_ref, unmodified reference sources) on the "
                    f"config's {wl.n_requests} requests ({wl.req_prompt[0]}+{wl.req_output[0]} "
                    f"tokens), {len(wl.chains)} tenants sharing the first "
                    f"{n_shared * s.n_layers} layers; prices blocks by cost tables, computes no "
                    "tensors",
            "batches": nb, "generated_tokens": rep.get("generated_tokens"),
            "simulated_tokens_per_s": rep.get("throughput_tokens_per_s"),
            "simulated_p95_latency_us": (rep.get("latency") or {}).get("p95_us")}


# ------------------------------------------------------------------------------------ GPU leg
def kernel_rooflines(ctx, wl, peaks):
    """Dominant kernels timed alone with CUDA events on the launching stream (inputs > L2)."""
    import numpy as np
    import torch
    from paper_2404_18322_b200 import device as dev
    from paper_2404_18322_b200._lib import lib, check
    import ctypes as C

    s = wl.shape
    stream = torch.cuda.ExternalStream(ctx.stream.value)
    res = {}
    # --- decode attention: 64 rows at ctx 640 over a 4-layer pool (671 MB of K/V per layer)
    rows, ctxlen, H, hd, L = 64, 640, s.n_heads, s.head_dim, s.n_layers
    pages_per_row = (ctxlen + 15) // 16
    n_pages = rows * pages_per_row
    blk_desc_shape = s
    blk = dev.Block(ctx, blk_desc_shape, "roofline", seed=3)
    pool = dev.KvPool(ctx, blk, n_pages)
    rng = np.random.default_rng(0)
    pt = rng.permutation(n_pages).astype(np.int32).reshape(rows, pages_per_row)
    d_pt = torch.from_numpy(pt).cuda()
    d_rowpt = torch.arange(rows, dtype=torch.int32, device="cuda")
    d_ctx = torch.full((rows,), ctxlen, dtype=torch.int32, device="cuda")
    q = torch.randn(rows, H * hd, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    torch.cuda.synchronize()

    def attn(layer):
        check(lib().be_attention(ctx.h, C.c_void_p(q.data_ptr()), C.c_void_p(pool.data_ptr), L, H,
                                 hd, layer, C.c_void_p(d_pt.data_ptr()), pages_per_row,
                                 C.c_void_p(d_rowpt.data_ptr()), C.c_void_p(d_ctx.data_ptr()),
                                 rows, 1, C.c_void_p(o.data_ptr()), C.c_void_p(0)), ctx.h)

    for layer in range(L):
        attn(layer)
    ctx.sync()
    reps = 8
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(reps):
        attn(i % L)
    e1.record(stream)
    ctx.sync()
    t = e0.elapsed_time(e1) / reps / 1e3
    bytes_ = rows * ctxlen * 2 * H * hd * 2 + 2 * rows * H * hd * 2
    res["attention"] = {"kernel": "attn_decode_kernel<128>", "shape": f"{rows} rows x ctx {ctxlen}, "
                        f"{H} heads x {hd}", "bytes_per_launch": bytes_, "us": t * 1e6,
                        "achieved_gbs": bytes_ / t / 1e9}
    pool.free()
    blk.free()

    # --- decode GEMMs at 64 rows, cycling through distinct weight copies (> L2)
    for name, N, K in [("gate_up", 2 * s.d_ff, s.d_model), ("qkv", 3 * s.d_model, s.d_model),
                       ("down", s.d_model, s.d_ff), ("o", s.d_model, s.d_model)]:
        copies = max(2, int(np.ceil(3 * 126e6 / (N * K * 2))))
        w = torch.empty(copies, N, K, dtype=torch.bfloat16, device="cuda").uniform_(-0.03, 0.03)
        for i in range(copies):
            w[i] = dev.pack_weight(ctx, w[i])
        x = torch.randn(64, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(64, N, device="cuda", dtype=torch.bfloat16)
        for i in range(copies):
            dev.gemm_bf16(ctx, w[i], x, out, packed=True)
        ctx.sync()
        reps = 4 * copies
        e0.record(stream)
        for i in range(reps):
            dev.gemm_bf16(ctx, w[i % copies], x, out, packed=True)
        e1.record(stream)
        ctx.sync()
        t = e0.elapsed_time(e1) / reps / 1e3
        bytes_ = 2 * (N * K + 64 * K + 64 * N)
        res[f"gemm_{name}"] = {"kernel": "gemm_tc_kernel<64>", "shape": f"[64x{K}]x[{K}x{N}]",
                               "bytes_per_launch": bytes_, "us": t * 1e6,
                               "achieved_gbs": bytes_ / t / 1e9,
                               "tflops": 2 * 64 * N * K / t / 1e12}
        del w
    torch.cuda.empty_cache()
    return res


def load_traffic():
    """ncu-measured DRAM bytes per launch by kernel family (profiles/ncu_traffic.json, written
    by scripts/ncu_traffic.py from one `ncu --set full` capture of a decode step), or {}."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def timeline_families(ctx, wl, fam_bytes):
    """The same decode step inside a CUDA-graph replay (PDL overlap included), timed by the
    kernels themselves (be_timeline_*: globaltimer at CTA start/end): each kernel is charged its
    marginal time, end(k) - end(k-1), so family times add up to the step. A separate runner
    (graphs are captured with the timeline slots in them); the context's timeline is off again
    afterwards."""
    from paper_2404_18322_b200.runner import Runner
    ctx.timeline_enable(4096)
    run = Runner(ctx, wl, mode=1, use_graphs=True)
    try:
        run.run()
        for _ in range(3):  # plain, capture, replay
            ctx.timeline_begin()
            run.decode_step()
            ctx.sync()
        recs = ctx.timeline_read()
    finally:
        run.close()
        ctx.timeline_enable(0)
    recs.sort(key=lambda r: r["end_last"])
    out, prev = {}, min(r["start_first"] for r in recs)
    for r in recs:
        f = "gemm" if r["cls"].startswith("gemm") else r["cls"]
        out[f] = out.get(f, 0.0) + max(0.0, (r["end_last"] - prev) / 1e3)
        prev = max(prev, r["end_last"])
    res = {}
    for f, us in out.items():
        b = fam_bytes.get(f)
        res[f] = {"us": round(us, 1), "achieved_gbs": round(b / (us / 1e6) / 1e9, 1) if b else None}
    return res


def profile_step(ctx, run, wl, stream, peaks, peaks_kind):
    """Per-launch event timing of one decode step; algorithmic bytes per launch:
    GEMM 2(NK + MK + MN); attention = the step's K/V bytes (runner accounting) + q and o rows;
    rms reads the fp32 residual; gather writes fp32 + bf16 rows; scatter copies bf16 rows."""
    import torch
    d = wl.shape.d_model
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ctx.sync()
    ctx.prof_enable(True)
    e0.record(stream)
    run.decode_step()
    e1.record(stream)
    recs = ctx.prof_read()
    ctx.prof_enable(False)
    step_ms = e0.elapsed_time(e1)
    st = run.step_stats()
    attn_rows = sum(r["ntok"] for r in recs if r["cls"] == "attention")
    fam = {}
    for r in recs:
        c, m, n, k = r["cls"], r["ntok"], r["n"], r["k"]
        if c.startswith("gemm"):
            b, fl, f = r["bytes"], r["flops"], "gemm"
        elif c == "attention":
            b = st["kv_bytes"] * m / max(1, attn_rows) + 2 * 2 * m * n * k
            fl, f = 0, "attention"
        elif c == "rms":
            b, fl, f = 4 * m * n, 0, "rms"
        elif c == "gather":
            b, fl, f = 8 * m * n, 0, "gather"
        else:
            b, fl, f = 4 * m * n, 0, "scatter"
        for key in (f, c) if f == "gemm" else (f,):
            a = fam.setdefault(key, {"launches": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0})
            a["launches"] += 1
            a["ms"] += r["ms"]
            a["bytes"] += b
            a["flops"] += fl
    hbm = peaks["hbm_gbs"]
    for a in fam.values():
        a["achieved_gbs"] = round(a["bytes"] / (a["ms"] / 1e3) / 1e9, 1) if a["ms"] else None
        a["frac"] = round(a["achieved_gbs"] / hbm, 4) if a["achieved_gbs"] else None
        a["share_of_step"] = round(a["ms"] / step_ms, 4)
        a["us_per_launch"] = round(1e3 * a["ms"] / a["launches"], 2)
        a["ms"] = round(a["ms"], 4)
    fam["_step"] = {"ms": round(step_ms, 4), "launches": len(recs),
                    "kernel_ms": round(sum(r["ms"] for r in recs), 4),
                    "note": "event-bracketed launches (no graph, no PDL overlap): the step here "
                            "is slower than a graph replay; shares are what matters"}
    top = max((k for k in fam if k in ("gemm", "attention", "rms", "gather", "scatter")),
              key=lambda k: fam[k]["ms"])
    a = fam[top]
    traffic = load_traffic().get(top)
    if traffic and abs(traffic.get("algorithmic_bytes_per_launch", 0) - a["bytes"] / a["launches"]) \
            > 0.01 * a["bytes"] / a["launches"]:
        traffic = None  # captured on another workload (the ncu capture is of C2's step)
    roofline = {"bound": "hbm", "kernel": {"gemm": "gemm_sk_kernel (all projections)",
                                           "attention": "attn_decode_kernel"}.get(top, top),
                "achieved": a["achieved_gbs"], "peak": hbm, "unit": "GB/s", "frac": a["frac"],
                "peak_kind": peaks_kind,
                "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                "traffic_algorithmic": round(a["bytes"] / a["launches"]),
                "traffic_source": traffic.get("source") if traffic else None,
                "launches_per_step": a["launches"], "us_per_launch": a["us_per_launch"],
                "share_of_step": a["share_of_step"],
                "tflops": round(a["flops"] / (a["ms"] / 1e3) / 1e12, 1) if a["flops"] else None}
    return {"roofline": roofline, "families": fam}


def make_workload(args, output=None):
    """The BASELINE config (configs[0..3] = c1..c4) at its own prompt / decode lengths unless
    --prompt / --output override them; `output` raises the decode length if a run needs more."""
    from paper_2404_18322_b200.workloads import CONFIGS
    kw = {}
    if args.prompt is not None and args.config != "c1":
        kw["prompt"] = args.prompt
    out = max(filter(None, [output, args.output])) if (output or args.output) else None
    if out is not None:
        kw["output"] = out
    return CONFIGS[args.config](**kw)


def run_pipeline(args, world, rank, local, depth, why):
    """N > 1 with chain positions cut into `depth` pipeline stages (world / depth replica groups
    side by side), `depth` micro-batches in flight per group, activation hops between stages by
    NCCL P2P over NVLink (paper_2404_18322_b200/pipeline.py)."""
    import torch
    import torch.distributed as dist
    from paper_2404_18322_b200.device import Context
    from paper_2404_18322_b200.pipeline import PipelineStage, ticks_needed, \
        tokens_per_request_needed

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    total = ticks_needed(depth, 2 * args.steps, args.warmup)  # device leg + end-to-end leg
    need = tokens_per_request_needed(depth, total, depth) + 1
    wl = make_workload(args, need)
    ctx = Context(local)
    group, st_idx = divmod(rank, depth)
    stage = PipelineStage(ctx, wl, depth, st_idx, base_rank=group * depth)
    clocks = ClockSampler(local)
    clocks.start()  # running long before the timed region; only its samples count
    t0 = time.time()
    stage.prefill()
    prefill_s = time.time() - t0
    warm = args.warmup + depth  # fill the pipeline
    for t in range(warm):
        stage.tick(t, total)
    ctx.sync()
    dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stage.stream)
    before = stage.stats.finished
    for t in range(warm, warm + args.steps):
        stage.tick(t, total)
    e1.record(stage.stream)
    ctx.sync()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    tm = torch.tensor([ms], device="cuda")
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms = float(tm.item())
    fin = torch.tensor([stage.stats.finished - before], device="cuda", dtype=torch.float64)
    dist.all_reduce(fin, op=dist.ReduceOp.SUM)  # only each group's last stage counts tokens
    tokens = float(fin.item())
    # end to end: stage 0 uploads each micro-batch's input rows from pinned host memory and the
    # last stage reads its output rows back every tick (decode_group host I/O)
    stage.set_host_io(True)
    if stage.host_in is not None:
        stage.host_in.copy_(torch.randn(stage.host_in.shape).to(torch.bfloat16))
    ctx.sync()
    dist.barrier()
    torch.cuda.synchronize()
    before = stage.stats.finished
    t_wall = time.perf_counter()
    e0.record(stage.stream)
    for t in range(warm + args.steps, warm + 2 * args.steps):
        stage.tick(t, total)
    e1.record(stage.stream)
    ctx.sync()
    torch.cuda.synchronize()
    e_ms = max(e0.elapsed_time(e1), (time.perf_counter() - t_wall) * 1e3)
    em = torch.tensor([e_ms], device="cuda")
    dist.all_reduce(em, op=dist.ReduceOp.MAX)
    ef = torch.tensor([stage.stats.finished - before], device="cuda", dtype=torch.float64)
    dist.all_reduce(ef, op=dist.ReduceOp.SUM)
    mb_bytes = stage.per_mb * wl.shape.d_model * 2
    e2e = {"value": round(float(ef.item()) / (float(em.item()) / 1e3), 2), "unit": "tokens/s",
           "h2d_bytes_per_step": mb_bytes, "d2h_bytes_per_step": mb_bytes,
           "ms_per_step": round(float(em.item()) / args.steps, 4)}
    stats = stage.run.step_stats()
    hop_bytes = wl.n_requests * wl.shape.d_model * 2
    if rank == 0:
        line = {
            "metric": "block-chain decode tokens/s", "value": round(tokens / (ms / 1e3), 2),
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": warm,
            "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, synthetic prompts; greedy feedback)",
            "config": {"workload": wl.name, "tenants": len(wl.chains),
                       "global_batch": wl.n_requests * world, "prompt": wl.req_prompt[0],
                       "decode": wl.req_output[0],
                       "parallelism": f"block placement: {world // depth} group(s) x {depth} "
                                      f"pipeline stages over chain positions {stage.stages}, "
                                      f"{depth} micro-batches of {wl.n_requests} per group, "
                                      f"NCCL P2P hops of {hop_bytes} B",
                       "placement": why,
                       "stage_cost_bytes": [round(c) for c in stage.stage_costs],
                       "l2": "inputs larger than L2"},
            "roofline": None, "e2e": e2e, "cpu_baseline": None,
            "gpu_launches": int(stats["launches"]) * args.steps, "clocks": clk,
            "prefill_s": round(prefill_s, 2),
            "note": "one step = one pipeline tick = one micro-batch token leaving each group's "
                    "last stage",
        }
        print(json.dumps(line), flush=True)
    stage.close()
    ctx.close()
    dist.destroy_process_group()


def time_steps(step, stream, steps, barrier):
    """Device time of `steps` calls of step() on `stream` (CUDA events, synchronised both
    sides), in ms, plus the host wall time."""
    import torch
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3


def run_cluster(args, world, rank, local):
    """N > 1 with block placement (paper_2404_18322_b200/cluster.py): every GPU holds the shared
    blocks and serves its own copy of the config's request mix (weak scaling); each tenant's
    private blocks live on the GPU choose_device(locality) picks and run all GPUs' rows for that
    tenant in one batch; rows hop there and back by NCCL send/recv (be_hop_*, one NCCL group per
    phase on the compute stream) inside the C++ executor loop (bh_cluster). The replica layout
    (every GPU holds every block, no hop) is measured in the same run for comparison."""
    import torch
    import torch.distributed as dist
    from paper_2404_18322_b200.cluster import Cluster, Comm, block_plan
    from paper_2404_18322_b200.device import Context
    from paper_2404_18322_b200.runner import Runner

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peaks_kind = load_peaks()
    wl = make_workload(args)
    d = wl.shape.d_model
    ctx = Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream.value)
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(Comm.unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    comm = Comm(ctx, world, rank, bytes(uid.cpu().numpy().tobytes()))
    plan = block_plan(wl, world)
    cl = Cluster({rank: ctx}, plan, comm, use_graphs=True, plan_ahead=True)
    clocks = ClockSampler(local)
    clocks.start()
    t0 = time.time()
    cl.prefill()
    ctx.sync()
    prefill_s = time.time() - t0
    home = cl.home(rank)
    n_live = home.live
    for _ in range(args.warmup):
        cl.decode_step()
    ctx.sync()

    def mx(v):
        t = torch.tensor([float(v)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    st0 = cl.stats()
    clocks.mark()
    ms, _ = time_steps(cl.decode_step, stream, args.steps, dist.barrier)
    clk = clocks.stop()
    st1 = cl.stats()
    ms = mx(ms)
    value = n_live * world * args.steps / (ms / 1e3)
    stats = cl.step_stats()
    step_bytes = stats["weight_bytes"] + stats["kv_bytes"] + stats["act_bytes"]
    step_bytes_max = mx(step_bytes)
    sent = (st1["sent_bytes"] - st0["sent_bytes"]) / args.steps
    recv = (st1["recv_bytes"] - st0["recv_bytes"]) / args.steps
    e2e = None
    if not args.no_e2e:
        hin = torch.randn(n_live, d).to(torch.bfloat16).pin_memory()
        hout = torch.empty(n_live, d, dtype=torch.bfloat16).pin_memory()
        cl.decode_step(hin, hout)
        bufs = [hin, hout]

        def e2e_step():
            cl.decode_step(bufs[0], bufs[1])
            bufs.reverse()  # greedy feedback: the step's output rows are the next input
        e_ms, wall = time_steps(e2e_step, stream, args.steps, dist.barrier)
        e_ms = mx(max(e_ms, wall))
        e2e = {"value": round(n_live * world * args.steps / (e_ms / 1e3), 2), "unit": "tokens/s",
               "h2d_bytes_per_step": int(hin.numel() * 2),
               "d2h_bytes_per_step": int(hout.numel() * 2),
               "ms_per_step": round(e_ms / args.steps, 4)}
    launches = int(stats["launches"])
    roofline = None
    if rank == 0 and not args.no_roofline:
        # the dominant kernel family of this rank's home runner (the shared blocks over its own
        # rows), one extra step of that runner with every launch bracketed by CUDA events; the
        # cluster is closed right after, so its desynchronised state is never used again
        try:
            home_wl = plan.runner(rank, 0).wl
            roofline = profile_step(ctx, home, home_wl, stream, peaks, peaks_kind)["roofline"]
            roofline["note"] = ("rank 0's home runner (shared blocks over its own rows): launches "
                                "bracketed by CUDA events on its stream (no graph, no PDL overlap)")
            roofline["traffic"] = None
            roofline["traffic_source"] = None
        except Exception as exc:  # diagnostics only
            roofline = {"error": str(exc)}
    cl.close()
    replicas = None
    if not args.no_replicas:
        run = Runner(ctx, wl, mode=1, use_graphs=True, plan_ahead=True)
        run.run()
        for _ in range(args.warmup):
            run.decode_step()
        ctx.sync()
        r_ms, _ = time_steps(run.decode_step, stream, args.steps, dist.barrier)
        r_ms = mx(r_ms)
        rst = run.step_stats()
        replicas = {"value": round(run.live * world * args.steps / (r_ms / 1e3), 2),
                    "ms_per_step": round(r_ms / args.steps, 4),
                    "bytes_per_step_per_gpu": rst["weight_bytes"] + rst["kv_bytes"]
                    + rst["act_bytes"],
                    "layout": "every GPU holds every block and serves its own request mix"}
        run.close()
    spec = None
    if args.spec or (args.spec is None and args.config == "c5"):
        spec = cluster_spec_leg(args, wl, plan, ctx, comm, world, rank, stream, mx)
    if rank == 0:
        hbm = peaks["hbm_gbs"]
        ms_step = ms / args.steps
        line = {
            "metric": "block-chain decode tokens/s", "value": round(value, 2), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, synthetic prompt embeddings; greedy "
                    "feedback of the last hidden state)",
            "config": run_config(wl, world),
            "config_detail": {"placement": plan.note, "processes": "one per GPU",
                              "hop_bytes_per_step_rank0": {"nccl_sent": sent,
                                                           "nccl_recv": recv}},
            "roofline": roofline,
            "step_roofline": {"bound": "hbm", "bytes_per_step_max_gpu": step_bytes_max,
                              "achieved": round(step_bytes_max / (ms_step / 1e3) / 1e9, 1),
                              "peak": hbm, "unit": "GB/s",
                              "frac": round(step_bytes_max / (ms_step / 1e3) / 1e9 / hbm, 4)},
            "replicas": replicas, "speculation": spec, "e2e": e2e, "cpu_baseline": None,
            "gpu_launches": launches * args.steps, "clocks": clk,
            "prefill_s": round(prefill_s, 2),
            "note": "gpu_launches: this rank's kernels (NCCL's send/recv kernels not counted)",
        }
        print(json.dumps(line), flush=True)
    comm.close()
    ctx.close()
    dist.destroy_process_group()


def cluster_spec_leg(args, wl, plan, ctx, comm, world, rank, stream, mx):
    """Speculative execution in the block-placed cluster (C5 = configs[4] on N GPUs): the blocks
    the reference's marking rule picks are shared blocks, present on every rank, so each rank's
    home runner drafts them with the 50%-FFN surrogate on its second stream, feeds the next block
    early and verifies with K7 on its own GPU; private blocks and hops as in the plain cluster.
    Tokens/s against the plain cluster step of the same run; accept counts summed over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2404_18322_b200.cluster import Cluster
    from paper_2404_18322_b200.pipeline import speculation_blocks
    blocks, marked = speculation_blocks(wl)
    out = {"marked_blocks": marked, "speculated_blocks": [wl.block_names[b] for b in blocks],
           "threshold": args.spec_threshold, "surrogate": "block with its FFN pruned to 50%"}
    if not blocks:
        out["note"] = "no marked block whose rows all continue to one block"
        return out
    cl = Cluster({rank: ctx}, plan, comm, use_graphs=True, spec_blocks=blocks,
                 spec_threshold=args.spec_threshold)
    try:
        cl.prefill()
        for _ in range(3):
            cl.decode_step()
        ctx.sync()
        n = cl.home(rank).live
        steps = max(3, min(args.steps, 10))
        ms, _ = time_steps(cl.decode_step, stream, steps, dist.barrier)
        ms = mx(ms)
        st = cl.spec_stats()
    finally:
        cl.close()
    t = torch.tensor([float(st["rows"]), float(st["accepted"]), float(st["cos_sum"])],
                     device="cuda", dtype=torch.float64)
    dist.all_reduce(t)
    rows, acc, cos_sum = (float(x) for x in t.tolist())
    out.update({"tokens_per_s": round(n * world * steps / (ms / 1e3), 2),
                "ms_per_step": round(ms / steps, 4), "steps": steps,
                "accept_rate": round(acc / rows, 4) if rows else None,
                "rows_verified_all_ranks": int(rows),
                "cos_mean": cos_sum / rows if rows else None,
                "note": "every rank drafts and verifies its own rows of the shared blocks on its "
                        "GPU; accept counts summed over ranks"})
    return out


def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    from paper_2404_18322_b200.device import Context
    from paper_2404_18322_b200.runner import Runner
    from paper_2404_18322_b200.workloads import CONFIGS

    placement = "1 GPU"
    if world > 1 and args.placement == "blocks":
        return run_cluster(args, world, rank, local)
    if world > 1:
        from paper_2404_18322_b200.pipeline import choose_layout
        lay = choose_layout(make_workload(args), world)
        depth = {"pipeline": world, "replica": 1, "auto": lay["depth"]}[args.placement]
        why = (f"{args.placement}: placement model picks depth {lay['depth']} x "
               f"{lay['replicas']} replicas (modelled max stage bytes/step "
               f"{world // lay['replicas'] / lay['score']:.3g}, stage HBM {lay['stage_mem']:.3g} B)")
        if depth > 1:
            return run_pipeline(args, world, rank, local, depth, why)
        placement = why
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peaks_kind = load_peaks()
    wl = make_workload(args)
    if world > 1:
        wl, routing = routed_share(wl, world, rank)
        placement += f"; {routing}"
    ctx = Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream.value)
    # plan_ahead: the host bookkeeping of step k+1 runs while step k is on the GPU (it matters
    # for the end-to-end leg, where each step waits for its output on the host)
    run = Runner(ctx, wl, mode=1, use_graphs=True, plan_ahead=True)
    clocks = ClockSampler(local)
    clocks.start()  # running long before the timed region; only its samples count
    t0 = time.time()
    run.run()  # prefill every prompt (untimed)
    ctx.sync()
    prefill_s = time.time() - t0
    n_live = run.live
    for _ in range(args.warmup):
        run.decode_step()
    ctx.sync()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # ---- device-timed region: K decode steps, inputs resident in HBM
    barrier()
    torch.cuda.synchronize()
    ctx.sync()
    clocks.mark()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if args.profile:
        torch.cuda.profiler.start()
    e0.record(stream)
    nb = 0
    for _ in range(args.steps):
        nb = run.decode_step()
    e1.record(stream)
    ctx.sync()
    torch.cuda.synchronize()
    if args.profile:
        torch.cuda.profiler.stop()
    clk = clocks.stop()
    barrier()
    ms = e0.elapsed_time(e1)
    stats = run.step_stats()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    tokens_per_step = n_live * world
    value = tokens_per_step * args.steps / (ms / 1e3)

    # ---- end to end through the public API: pinned host rows in, results out, every step
    e2e = None
    if not args.no_e2e:
        d = wl.shape.d_model
        hin = torch.empty(n_live, d, dtype=torch.bfloat16).pin_memory()
        hout = torch.empty(n_live, d, dtype=torch.bfloat16).pin_memory()
        hin.copy_(torch.randn(n_live, d).to(torch.bfloat16))
        run.decode_step(hin, hout)
        barrier()
        ctx.sync()
        t_start = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            run.decode_step(hin, hout)
            hin, hout = hout, hin  # greedy feedback: the step's output buffer is the next input
        e1.record(stream)
        ctx.sync()
        wall = time.perf_counter() - t_start
        e_ms = max(e0.elapsed_time(e1), wall * 1e3)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": tokens_per_step * args.steps / (e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(hin.numel() * 2), "d2h_bytes_per_step": int(hout.numel() * 2),
               "ms_per_step": e_ms / args.steps}

    # ---- roofline: one more decode step with every launch bracketed by CUDA events on the
    # runner's stream (graph replay bypassed for this step only), kernels grouped by family
    prof = profile_step(ctx, run, wl, stream, peaks, peaks_kind) if not args.no_roofline else None
    roofline = prof["roofline"] if prof else None
    if prof is not None and world == 1:
        # the same kernels inside the graph-replayed step (marginal in-step time per family)
        fam_bytes = {k: v["bytes"] for k, v in prof["families"].items() if isinstance(v, dict)
                     and "bytes" in v}
        try:
            tl = timeline_families(ctx, wl, fam_bytes)
            prof["families"]["_in_step_timeline"] = tl
            tl["note"] = ("diagnostics: a separate runner's graph-replayed step timed by the "
                          "kernels' own globaltimer stamps (marginal time per kernel); its "
                          "families do not sum to the bench step (other clocks, timeline "
                          "slots in the graph), so the roofline above uses the event-bracketed "
                          "launches")
            roofline["note"] = ("achieved: the family's launches bracketed by CUDA events on "
                                "the runner's stream (one extra step, no graph, no PDL overlap)")
        except Exception as exc:  # diagnostics only
            msg = str(exc)
            prof["families"]["_in_step_timeline"] = (
                {"skipped": "a second runner of this config does not fit beside the measured one"}
                if "out of device memory" in msg else {"error": msg})
    kr = kernel_rooflines(ctx, wl, peaks) if rank == 0 and args.isolated else {}
    live = spec = None
    if world == 1 and not args.no_live:
        run.close()  # the live runner loads its own copy of the zoo
        live = live_leg(ctx, args, wl)
    if world == 1 and (args.spec or (args.spec is None and args.config == "c5")):
        run.close()
        spec = spec_leg(ctx, args, wl, peaks, stream)
    hbm = peaks["hbm_gbs"]
    step_bytes = stats["weight_bytes"] + stats["kv_bytes"] + stats["act_bytes"]
    step_roofline = {"bound": "hbm", "bytes_per_step": step_bytes,
                     "achieved": round(step_bytes / (ms_per_step / 1e3) / 1e9, 1), "peak": hbm,
                     "unit": "GB/s", "frac": round(step_bytes / (ms_per_step / 1e3) / 1e9 / hbm, 4),
                     "roofline_tokens_per_s": round(n_live * hbm * 1e9 / step_bytes, 1)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        cs = CpuDecodeStep(wl, threads)
        cs.step()  # first touch
        t_step = cs.step()
        cpu = {"value": round(n_live / t_step, 3), "unit": "tokens/s", "cores": threads,
               "kind": "port", "sample": cs.sample() + f" ({t_step:.2f} s)",
               "reference_sim": blocksim_run(wl)}
        del cs

    if rank == 0:
        line = {
            "metric": "block-chain decode tokens/s", "value": round(value, 2), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, "
            "synthetic prompt embeddings; greedy feedback of the last hidden state)",
            "config": run_config(wl, world),
            "config_detail": {"model": {"c1": "tiny decoder", "c2": "Llama-2-7B-shaped",
                                        "c3": "Llama-2-7B-shaped", "c4": "Llama-2-13B-shaped",
                                        "c5": "Llama-2-7B-shaped",
                                        "c2lora": "Llama-2-7B-shaped + rank-16 LoRA tenants"
                                        }.get(args.config, wl.name),
                              "batches_per_step": nb,
                              "parallelism": f"replica per GPU x{world}" if world > 1 else "1 GPU",
                              "placement": placement},
            "roofline": roofline, "step_roofline": step_roofline,
            "kernels": prof["families"] if prof else None,
            "kernels_isolated": kr or None,
            "latency": live, "speculation": spec,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(stats["launches"]) * args.steps,
            "graph_replayed": bool(stats["graph_replayed"]), "clocks": clk,
            "prefill_s": round(prefill_s, 2),
        }
        print(json.dumps(line), flush=True)
    run.close()
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def routed_share(wl, world, rank):
    """Replica placement: the global stream is `world` copies of the config's requests; each
    request binds to a replica through bh_policy_choose_binding (the reference's estimate rule,
    priced by the measured B200 profiles) and stays there for decode (KV owner). Returns this
    rank's share as a workload, plus a note for the JSON line."""
    import dataclasses
    from paper_2404_18322_b200.pipeline import route_requests
    dev = route_requests(wl, world, copies=world)
    mine = [g // world for g, d in enumerate(dev) if d == rank]
    share = dataclasses.replace(wl, req_tenant=[wl.req_tenant[i] for i in mine],
                                req_prompt=[wl.req_prompt[i] for i in mine],
                                req_output=[wl.req_output[i] for i in mine])
    counts = [dev.count(r) for r in range(world)]
    return share, f"requests routed by bh_policy choose_binding: {counts} per replica"


def run_reference(args, world, rank, local):
    """The reference arm: the path's arithmetic on the host cores, whole decode steps. The
    reference computes no tensors (blocksim prices a block with CostModel::block_us), so the
    timed CPU implementation is the oracle port of the block forward (CpuDecodeStep: every block
    run of a step, all host threads); blocksim's own Simulation::run on the same requests is
    reported beside it (reference_sim)."""
    if rank != 0:
        return
    wl = make_workload(args)
    threads = os.cpu_count() or 1
    cs = CpuDecodeStep(wl, threads)
    t_wall = time.perf_counter()
    for _ in range(args.warmup):
        cs.step()
    times = [cs.step() for _ in range(args.steps)]
    wall = time.perf_counter() - t_wall
    ms_step = 1e3 * sum(times) / len(times)
    v = wl.n_requests / (ms_step / 1e3)
    sim = blocksim_run(wl)
    line = {"impl": "reference", "metric": "block-chain decode tokens/s", "value": round(v, 3),
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": run_config(wl, world),
            "cpu_baseline": {"value": round(v, 3), "unit": "tokens/s", "cores": threads,
                             "kind": "port", "sample": cs.sample(),
                             "timed_wall_s": round(wall, 2), "reference_sim": sim},
            "e2e": {"value": round(v, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def live_leg(ctx, args, wl):
    """p95 request latency (BASELINE.json metric): the config's request mix (2x its requests,
    tenants round-robin) arriving as a Poisson process at --qps, served live by one runner
    (bh_runner_serve: arrivals prefilled as they come, then boarding the next lockstep decode
    iteration); latency = completion - arrival, ttft = first token - arrival, nearest-rank
    percentiles and tokens / drain time as the reference reports them (metrics.cpp:30-38,
    159-190). Wall-clock time stamps on the host after the device finished each token."""
    import dataclasses
    from paper_2404_18322_b200.metrics import poisson_arrivals, serving_report
    from paper_2404_18322_b200.runner import Runner
    n = args.live_requests or 2 * wl.n_requests
    # every live request holds full-length KV in every block of its chain: stay within HBM
    per_req = max(len(c) for c in wl.chains) * (wl.req_prompt[0] + wl.req_output[0] + 32) \
        * wl.shape.kv_bytes_per_token
    weights = len(wl.block_names) * wl.shape.param_bytes
    while n > wl.n_requests and weights + n * per_req > 140e9:
        n -= wl.n_requests
    T = len(wl.chains)
    out = wl.req_output[0] if args.output is None else min(wl.req_output[0], 128)
    lw = dataclasses.replace(wl, req_tenant=[i % T for i in range(n)],
                             req_prompt=[wl.req_prompt[0]] * n, req_output=[out] * n)
    arr = poisson_arrivals(n, args.qps, seed=wl.seed)
    run = Runner(ctx, lw, mode=1, use_graphs=True)
    try:
        first, done = run.serve(arr)
        rep = serving_report(arr, first, done, run.tokens_generated)
    finally:
        run.close()
    rep.update({"qps": args.qps, "arrivals": f"Poisson, seed {wl.seed}",
                "prompt": lw.req_prompt[0], "output": out,
                "scheduling": "arrivals prefilled on arrival (token budget "
                              f"{wl.max_batch_tokens}), then join the next lockstep decode step"})
    return rep


def k7_roofline(ctx, rows, d, peaks):
    """K7 (the cosine verdict kernel, be_cosine) timed alone at the speculative batch size:
    algorithmic bytes 2 * rows * d * 2 (both bf16 inputs read once) per launch, launches cycling
    over 32 input pairs (> L2), CUDA events on the launching stream."""
    import torch
    from paper_2404_18322_b200 import device as dev
    stream = torch.cuda.ExternalStream(ctx.stream.value)
    pairs = [(torch.randn(rows, d, device="cuda").to(torch.bfloat16),
              torch.randn(rows, d, device="cuda").to(torch.bfloat16)) for _ in range(32)]
    cos = torch.empty(rows, device="cuda")
    acc = torch.empty(rows, device="cuda", dtype=torch.int32)
    for a, b in pairs[:4]:
        dev.cosine(ctx, a, b, 0.95, cos, acc)
    ctx.sync()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = 128
    e0.record(stream)
    for i in range(reps):
        a, b = pairs[i % 32]
        dev.cosine(ctx, a, b, 0.95, cos, acc)
    e1.record(stream)
    ctx.sync()
    us = e0.elapsed_time(e1) * 1e3 / reps
    byts = 2 * rows * d * 2
    return {"kernel": "cosine_rows_kernel (K7)", "shape": f"{rows} rows x {d}", "bound": "hbm",
            "us_per_launch": round(us, 2), "bytes_per_launch": byts,
            "achieved": round(byts / (us * 1e-6) / 1e9, 1), "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": round(byts / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 4),
            "note": "a 4 MB launch is latency-bound: the verdict costs a few us per speculative "
                    "block run"}


def spec_leg(ctx, args, wl, peaks, stream):
    """Speculative execution inside the lockstep executor loop: the blocks the
    reference's marking rule picks (pipeline.speculation_blocks = bh_policy_speculation_marks)
    run with their 50%-FFN surrogate on a second stream feeding the next block early, K7
    (cosine >= threshold) accepting rows, rejected rows re-running the next block. Tokens/s
    with speculation against the plain step of the same runner, accept rate, K7 roofline."""
    from paper_2404_18322_b200.pipeline import speculation_blocks
    from paper_2404_18322_b200.runner import Runner
    blocks, marked = speculation_blocks(wl)
    out = {"marked_blocks": marked,
           "speculated_blocks": [wl.block_names[b] for b in blocks],
           "threshold": args.spec_threshold, "surrogate": "block with its FFN pruned to 50%"}
    if not blocks:
        out["note"] = "no marked block whose rows all continue to one block"
        return out
    run = Runner(ctx, wl, mode=1, use_graphs=True, spec_blocks=blocks,
                 spec_threshold=args.spec_threshold)
    try:
        run.run()
        for _ in range(3):
            run.decode_step()
        ctx.sync()
        n = run.live
        steps = max(3, min(args.steps, 10))
        ms, _ = time_steps(run.decode_step, stream, steps, lambda: None)
        st = run.spec_stats()
    finally:
        run.close()
    rows = max(wl.rows_at_block()[b] for b in blocks)
    out.update({"tokens_per_s": round(n * steps / (ms / 1e3), 2),
                "ms_per_step": round(ms / steps, 4), "steps": steps,
                "accept_rate": round(st["accept_rate"], 4) if st["accept_rate"] is not None
                else None, "rows_verified": st["rows"],
                "cos_mean": st["cos_mean"], "cos_min": st["cos_min"],
                "k7": k7_roofline(ctx, rows, wl.shape.d_model, peaks),
                "note": "one GPU: draft and verify share its SMs and HBM, so the speculative step "
                        "streams the surrogate's weights on top of the block's - slower; the "
                        "paper's gain needs the next block on another GPU"})
    return out


def run_config(wl, world):
    """The `config` object of a bench line (both arms): the workload and its shape."""
    return {"workload": wl.name, "tenants": len(wl.chains), "global_batch": wl.n_requests * world,
            "prompt": wl.req_prompt[0], "decode": wl.req_output[0],
            "blocks": f"{len(wl.block_names)} blocks x {wl.shape.n_layers} layers",
            "rows_per_block": wl.rows_at_block(),
            "parallelism": "1 GPU" if world == 1 else f"block placement over {world} GPUs",
            "l2": "inputs larger than L2 (weights+KV streamed per step)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "c2lora"])
    ap.add_argument("--prompt", type=int, default=None, help="default: the config's own")
    ap.add_argument("--output", type=int, default=None, help="default: the config's own")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--placement", default="blocks",
                    choices=["blocks", "auto", "pipeline", "replica"],
                    help="N>1: block placement (shared blocks on every GPU, private blocks by "
                         "choose_device, NCCL hops; default), the position-pipeline model's "
                         "choice (auto), chain positions cut into N pipeline stages, or one "
                         "replica of the zoo per GPU")
    ap.add_argument("--no-live", action="store_true", help="skip the live p95-latency leg")
    ap.add_argument("--spec", dest="spec", action="store_true", default=None,
                    help="add the speculative-execution leg (default: on for --config c5)")
    ap.add_argument("--no-spec", dest="spec", action="store_false")
    ap.add_argument("--spec-threshold", type=float, default=0.95)
    ap.add_argument("--qps", type=float, default=32.0,
                    help="live leg: Poisson arrival rate (requests/s)")
    ap.add_argument("--live-requests", type=int, default=None,
                    help="live leg: requests (default 2x the config's)")
    ap.add_argument("--no-replicas", action="store_true",
                    help="N>1 block placement: skip the replica comparison leg")
    ap.add_argument("--isolated", action="store_true",
                    help="also time the dominant kernels alone (standalone launches, > L2)")
    ap.add_argument("--profile", action="store_true",
                    help="cudaProfilerStart/Stop around the timed steps (ncu --profile-from-start off)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup()
    need = 1 + args.warmup + 2 * args.steps + 2  # value leg + e2e leg + the profiled steps
    if make_workload(args).req_output[0] < need:
        args.output = need
    if args.impl == "reference":
        run_reference(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
