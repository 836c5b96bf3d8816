#!/usr/bin/env python3
"""FCP block-attention fwd+bwd benchmark on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

A step = one attention layer forward + backward over the whole batch: FCP plan
(computed once per batch, outside the timed region, like the paper) -> per rank:
local tiles, staged KV exchange over NVLink overlapped with released tiles,
LSE merge, backward with the dK/dV return.  Prints ONE JSON line on rank 0.

Metric (BASELINE.json): CP attention fwd+bwd tokens/s (sum of sequence lengths /
max-over-ranks step time) and MFU = 3.5 * 4*Hq*D*sum L(L+1)/2 / (N * peak * T).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2605_08524_b200 import configs  # noqa: E402
from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY, batch_token_pairs  # noqa: E402
from paper_2605_08524_b200.distributor import worker_loads  # noqa: E402
from paper_2605_08524_b200.pipeline import fcp_schedule, plan_digest  # noqa: E402
from paper_2605_08524_b200.sharding import ShardingConfig  # noqa: E402

METRIC = "CP attention fwd+bwd tokens/sec and MFU at 1/2/4/8 B200 (max over ranks)"
UNIT = "tokens/s"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["bf16_tflops"]) * 1e12, float(d.get("bf16_tflops_sustained", 0)) * 1e12, \
            float(d.get("hbm_gbs", 6555)) * 1e9, "measured"
    except Exception:
        return 1.59e15, 1.4e15, 6.65e12, "fallback"


class ClockSampler:
    """SM clock, power and clock-event reasons sampled through NVML every 20 ms during the
    timed region (nvidia-smi as the fallback), plus the NVML energy counter around it."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int):
        self.index = index
        self.samples = []          # (sm_mhz, power_w, reasons bitmask)
        self._stop = threading.Event()
        self._t = None
        self.nv = None
        self.energy_mj = None
        try:
            import pynvml
            pynvml.nvmlInit()
            # CUDA_VISIBLE_DEVICES may remap; the bench process sees its GPU as `index`
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[index]) if vis and vis.split(",")[index].isdigit() else index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1e3
        except Exception:
            self.nv = None

    def _energy(self):
        try:
            return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h)
        except Exception:
            return None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                if nv is not None:
                    self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                         nv.nvmlDeviceGetPowerUsage(self.h) / 1e3,
                                         nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
                else:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,power.draw",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip()
                    if out:
                        sm, pw = (float(x) for x in out.split(",")[:2])
                        self.samples.append((sm, pw, 0))
            except Exception:
                pass
            self._stop.wait(0.02 if nv is not None else 0.2)

    def __enter__(self):
        e0 = self._energy() if self.nv else None
        self._e0 = e0
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)
        if self.nv and self._e0 is not None:
            e1 = self._energy()
            self.energy_mj = None if e1 is None else e1 - self._e0

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = sorted(x[0] for x in self.samples)
        reasons = []
        if self.nv is not None:
            for name, attr in self.REASONS:
                bit = getattr(self.nv, attr, 0)
                if bit and any(x[2] & bit for x in self.samples):
                    reasons.append(name)
        out = {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": getattr(self, "max_mhz", None),
               "reasons": reasons, "samples": len(self.samples), "sm_mhz_min": sm[0]}
        if self.nv is not None:
            out["power_limit_w"] = self.limit_w
        return out


def measured_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the committed
    ncu --set full summary (profiles/traffic.json, scripts/ncu_summary.py); None if absent."""
    try:
        d = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                        "traffic.json")))
        k = d["kernels"][kernel]
        return {"bytes_per_launch": k["traffic_bytes"], "source": d["source"]}
    except Exception:
        return None


def build_workload(name: str, n: int, block: int | None, scheduler: str = "fcp",
                   curve: str = "reference"):
    """The workload and its plan: FCP (default), or the reference's competitor plans
    (ring / ByteScale) executed by the same B200 executor."""
    w = configs.by_name(name, n, block)
    if scheduler == "ring":
        from paper_2605_08524_b200.baselines import ring_schedule
        return w, ring_schedule(w.batch(), n, w.model)
    if scheduler == "bytescale":
        from paper_2605_08524_b200.baselines import bytescale_schedule
        return w, bytescale_schedule(w.batch(), n, w.tokens_per_worker, w.model)
    from paper_2605_08524_b200.costmodel import B200_EFFICIENCY
    result = fcp_schedule(w.batch(), n, ShardingConfig(block_size=w.block_size), w.model,
                          B200_EFFICIENCY if curve == "b200" else DEFAULT_EFFICIENCY)
    return w, result


def rank_inputs(ex, rank, cfg, device, pin=False):
    """Q, K, V, dO ~ N(0,1) rounded to bf16, drawn on the device from a generator seeded
    1234 + rank; pinned host copies only when the e2e leg needs them."""
    g = torch.Generator(device=device).manual_seed(1234 + rank)
    T, H, Hk, D = ex.tokens, cfg.q_heads, cfg.kv_heads, cfg.head_dim
    dev = [torch.randn((T, h, D), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
           for h in (H, Hk, Hk, H)]
    host = [x.cpu().pin_memory() for x in dev] if pin else None
    return host, dev


def e2e_sequential(ex, host, device, steps, barrier):
    """Median wall time of one fully serial step: H2D of the inputs, fwd+bwd, D2H of all
    outputs, synchronised on both sides."""
    ts = []
    for it in range(steps + 1):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        qd, kd, vd, dod = (x.to(device, non_blocking=True) for x in host)
        res = [t.to("cpu", non_blocking=True) for t in ex.step(qd, kd, vd, dod)]
        torch.cuda.synchronize()
        if it:
            ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2]


def e2e_pipelined(ex, host, device, steps, warmup, barrier):
    """Per-step wall time of a pipelined loop through the public executor API.  Every step
    copies its own Q/K/V/dO from pinned host memory and its O, LSE, dQ, dK, dV back to
    pinned host memory; the copies run on two copy streams so that dO lands during the
    forward, O/LSE leave during the backward, and step i+1's inputs arrive while step i's
    gradients leave (inputs double-buffered on the device).  Returns (s/step, D2H bytes)."""
    cur = torch.cuda.current_stream(device)
    s_in, s_out = torch.cuda.Stream(device=device), torch.cuda.Stream(device=device)
    bufs = [[torch.empty_like(x, device=device) for x in host] for _ in range(2)]
    freed = [None, None]                  # event: compute of the step that used the buffer
    outs_host = [None, None]
    d2h = 0

    def run(n):
        nonlocal d2h
        for it in range(n):
            b = it & 1
            q, k, v, do = bufs[b]
            with torch.cuda.stream(s_in):
                if freed[b] is not None:
                    s_in.wait_event(freed[b])
                for dst, src in zip((q, k, v), host[:3]):
                    dst.copy_(src, non_blocking=True)
                ev_qkv = torch.cuda.Event()
                ev_qkv.record(s_in)
                do.copy_(host[3], non_blocking=True)
                ev_do = torch.cuda.Event()
                ev_do.record(s_in)
            cur.wait_event(ev_qkv)
            o, lse = ex.forward(q, k, v)
            ev_f = torch.cuda.Event()
            ev_f.record(cur)
            cur.wait_event(ev_do)
            dq, dk, dv = ex.backward(q, k, v, o, lse, do)
            ev_b = torch.cuda.Event()
            ev_b.record(cur)
            freed[b] = ev_b
            outs = (o, lse, dq, dk, dv)
            if outs_host[b] is None:
                outs_host[b] = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs]
                d2h = sum(t.numel() * t.element_size() for t in outs)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_f)
                for hst, t in zip(outs_host[b][:2], outs[:2]):
                    hst.copy_(t, non_blocking=True)
                s_out.wait_event(ev_b)
                for hst, t in zip(outs_host[b][2:], outs[2:]):
                    hst.copy_(t, non_blocking=True)
            for t in outs:                    # keep the caching allocator off them until copied
                t.record_stream(s_out)

    run(max(warmup, 2))
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    run(steps)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    return dt, d2h


# ---------------------------------------------------------------------------- CPU legs
def cpu_model() -> str:
    """The host CPU model (lscpu's 'Model name'), recorded next to the CPU numbers."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample_unit(result):
    """The fixed CPU sample: the schedule unit (zigzag pair) that holds the first and the last
    chunk of the batch's longest sequence, i.e. its diagonal-only chunk and its chunk with the
    longest KV list (reference ``sharding.py:84-88,172-201``).  Returns (seq_len, [(q_start,
    q_len, kv_len, diag_from)], visible pairs)."""
    from paper_2605_08524_b200.costmodel import tile_token_pairs
    deps = result.deps
    seq_len: dict[int, int] = {}
    for (sid, _), n in deps.chunk_tokens.items():
        seq_len[sid] = seq_len.get(sid, 0) + n
    sid = max(seq_len, key=lambda s_: (seq_len[s_], -s_))
    unit = next(u for u in result.units if any(m.key == (sid, 0) for m in u.members))
    starts: dict = {}
    pos = 0
    for key in sorted((kk for kk in deps.chunk_tokens if kk[0] == sid), key=lambda kk: kk[1]):
        starts[key] = pos
        pos += deps.chunk_tokens[key]
    parts, pairs = [], 0
    for m in unit.members:
        kvs = deps.q_to_kv[m.key]
        q0, qn = starts[m.key], m.token_count
        kv_len = sum(deps.chunk_tokens[kv] for kv in kvs)
        parts.append((q0, qn, kv_len, kv_len - qn))
        pairs += sum(tile_token_pairs(qn, deps.chunk_tokens[kv], kv == m.key) for kv in kvs)
    return seq_len[sid], parts, pairs


def cpu_sample(w, result, reps=1, threads=None):
    """Oracle fp32 fwd+bwd (torch CPU, all host threads) of the fixed sample of
    ``cpu_sample_unit``; tokens/s of the whole batch extrapolated by its pair fraction.
    The same sample in both CPU legs (this arm's ``cpu_baseline`` and ``--impl reference``).
    Returns ([tokens/s per rep], info)."""
    sys.path.insert(0, ROOT)
    from oracle.attention_ref import chunk_fwd_bwd
    threads = threads or os.cpu_count()
    torch.set_num_threads(threads)
    cfg = w.model
    L, parts, pairs = cpu_sample_unit(result)
    g = torch.Generator().manual_seed(1234)
    mk = lambda h: torch.randn((L, h, cfg.head_dim), generator=g).to(torch.bfloat16).float()
    q, k, v, do = mk(cfg.q_heads), mk(cfg.kv_heads), mk(cfg.kv_heads), mk(cfg.q_heads)
    scale = 1.0 / math.sqrt(cfg.head_dim)
    total_pairs = batch_token_pairs(list(w.lengths), "causal")
    vals = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for q0, qn, kv_len, diag_from in parts:
            chunk_fwd_bwd(q, k, v, do, torch.arange(q0, q0 + qn), torch.arange(kv_len), diag_from, scale)
        dt = time.perf_counter() - t0
        vals.append(w.total_tokens / (dt * total_pairs / pairs))
    info = {"cores": threads, "cpu_model": cpu_model(), "pair_fraction": pairs / total_pairs,
            "sample": (f"oracle fp32 fwd+bwd (torch CPU, {threads} threads) of the zigzag unit holding "
                       f"the first and last chunk of the longest sequence (L={L}: Q chunks "
                       f"{[(p[1], p[2]) for p in parts]} as (q rows, kv rows)) = {pairs} visible pairs, "
                       f"{pairs / total_pairs:.4f} of the batch's; tokens/s extrapolated by pair count")}
    return vals, info


def workload_config(w, n, scheduler="fcp"):
    """The `config` dict both arms print (identical keys and values)."""
    return {"workload": w.name, "global_batch_tokens": w.total_tokens, "sequences": len(w.lengths),
            "block": w.block_size, "q_heads": w.model.q_heads, "kv_heads": w.model.kv_heads,
            "head_dim": w.model.head_dim, "parallelism": f"{scheduler}{n}",
            "l2": "inputs larger than L2 (no flush needed)"}


def reference_control_plane(w, n):
    """The reference's own fcp_schedule (unmodified, baseline/_ref) on 1 core."""
    sys.path.insert(0, ROOT)
    from oracle import ref_control_plane
    m = w.model
    return ref_control_plane.run(w.lengths, n, w.tokens_per_worker, w.block_size,
                                 dict(q_heads=m.q_heads, kv_heads=m.kv_heads, head_dim=m.head_dim,
                                      dtype_bytes=m.dtype_bytes))


def run_reference(args):
    """--impl reference: the reference path's CPU implementation on the box's host cores.
    The reference has no attention code, so the attention math is the oracle port
    (fp32, all host threads, the fixed sample of ``cpu_sample_unit`` per step); the reference's
    own control plane (``fcp_schedule`` from baseline/_ref, 1 core) is timed beside it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.gpus
    w, result = build_workload(args.config, n, args.block, args.scheduler)
    vals, info = cpu_sample(w, result, reps=args.warmup + args.steps)
    vals = vals[args.warmup:]
    value = sorted(vals)[len(vals) // 2]
    t_step = w.total_tokens / value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong" if args.config in ("c2", "c3") else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(w, n, args.scheduler),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "port",
                             "cpu_model": info["cpu_model"], "sample": info["sample"],
                             "spread": [min(vals), max(vals)]},
            "reference_control_plane": reference_control_plane(w, n),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--block", type=int, default=None)
    ap.add_argument("--scheduler", default="fcp", choices=["fcp", "ring", "bytescale"],
                    help="plan to execute (ring / bytescale: the reference's competitors)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # The reference's planner takes its efficiency curve as an input (costmodel.py:63-127).
    # The headline plans with the reference's stock DEFAULT_EFFICIENCY; the curve
    # measured on B200 (costmodel.B200_EFFICIENCY) is a labelled variant, its plans pinned to
    # the unmodified reference run with the same anchors
    # (tests/test_plan_parity.py::test_plan_bit_identical_with_b200_curve).
    ap.add_argument("--curve", default="reference", choices=["reference", "b200"],
                    help="efficiency curve the LPT placement plans with (costmodel.py)")
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = world if world > 1 else args.gpus
    if world == 1 and args.gpus > 1:
        # not launched under torchrun: N independent ranks need N processes
        raise SystemExit("run N>1 under torch.distributed.run (one process per GPU)")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    from paper_2605_08524_b200.executor import FcpExecutor

    peak, peak_sus, hbm, peak_kind = load_peaks()
    w, result = build_workload(args.config, n, args.block, args.scheduler, args.curve)
    # host control plane (fcp_schedule), median of 5 warm calls -- the same statistic as
    # the reference's own fcp_schedule timed beside it (oracle/ref_control_plane.py)
    from paper_2605_08524_b200.costmodel import B200_EFFICIENCY
    plan_ts = []
    batch = w.batch()
    for _ in range(5):
        t_plan = time.perf_counter()
        fcp_schedule(batch, n, ShardingConfig(block_size=w.block_size), w.model,
                     B200_EFFICIENCY if args.curve == "b200" else DEFAULT_EFFICIENCY)
        plan_ts.append((time.perf_counter() - t_plan) * 1e3)
    plan_ms = sorted(plan_ts)[2]
    cfg = w.model
    ex = FcpExecutor(result, rank, cfg, device)
    host, (q, k, v, do) = rank_inputs(ex, rank, cfg, device, pin=not args.no_e2e)
    # K/V live in the executor's input buffers (at N > 1 the exchange region's K/V planes,
    # which the peers read in place: no per-step publish copy)
    kb, vb = ex.kv_input_buffers()
    kb.copy_(k)
    vb.copy_(v)
    k, v = kb, vb
    stream = torch.cuda.current_stream(device)

    # kernel-level events (on the launching stream) for the roofline
    lib_launch = {"fwd": [], "bwd": [], "dq": []}
    orig_fw, orig_bl, orig_dq = ex.op.forward_wave, ex.op.backward_launch, ex.op.backward_dq
    timing = {"on": False}

    def timed_fw(*a, **kw):
        if not timing["on"]:
            return orig_fw(*a, **kw)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        orig_fw(*a, **kw)
        e.record(stream)
        lib_launch["fwd"].append((s, e))

    def timed_bl(recv, *a, **kw):
        if not timing["on"]:
            return orig_bl(recv, *a, **kw)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        orig_bl(recv, *a, **kw)
        e.record(stream)
        lib_launch["bwd"].append((s, e))

    def timed_dq(*a, **kw):
        if not timing["on"]:
            return orig_dq(*a, **kw)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        out = orig_dq(*a, **kw)
        e.record(stream)
        lib_launch["dq"].append((s, e))
        return out

    ex.op.forward_wave, ex.op.backward_launch, ex.op.backward_dq = timed_fw, timed_bl, timed_dq

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        ex.step(q, k, v, do)
    torch.cuda.synchronize()
    barrier()
    launches0 = ex.op.launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            ex.step(q, k, v, do)
        end.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = ex.op.launches - launches0
    ms = start.elapsed_time(end) / args.steps
    # Energy per step: the NVML energy counter needs a window of about a second, so it is read
    # over a separate untimed loop of at least 1.5 s (the timed region may be shorter).
    energy = None
    # every rank must run the same number of steps (the exchange's flag barriers are
    # collective): size the loop from the max-over-ranks step time
    t_e = torch.tensor([ms], device=device)
    if world > 1:
        dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
    e_steps = max(args.steps, int(math.ceil(1500.0 / max(t_e.item(), 1e-3))))
    with ClockSampler(local) as eclk:
        torch.cuda.synchronize()
        for _ in range(e_steps):
            ex.step(q, k, v, do)
        torch.cuda.synchronize()
    if eclk.energy_mj is not None and eclk.energy_mj > 0:
        energy = {"j_per_step": round(eclk.energy_mj / 1e3 / e_steps, 3),
                  "power_w_avg": round(eclk.energy_mj / (e_steps * ms), 1), "steps": e_steps,
                  "window_s": round(e_steps * ms / 1e3, 2),
                  "how": "NVML total-energy counter over a separate untimed loop of >= 1.5 s"}
    # per-kernel share (separate pass so the kernel events do not perturb the step time)
    timing["on"] = True
    for _ in range(min(3, args.steps)):
        ex.step(q, k, v, do)
    torch.cuda.synchronize()
    timing["on"] = False
    ex.timeline(True)
    for _ in range(3):
        ex.step(q, k, v, do)
    phases = ex.phases()
    ex.timeline(False)
    phases_all = None
    if world > 1:               # every rank's timeline: who waits for whom at the barriers
        phases_all = [None] * world
        dist.all_gather_object(phases_all, {kk: round(vv, 3) for kk, vv in phases.items()})
    # e2e: host buffers in, results out, through the public executor API
    e2e = None
    if not args.no_e2e:
        h2d = sum(x.numel() * x.element_size() for x in host)
        seq_s = e2e_sequential(ex, host, device, min(args.steps, 5), barrier)
        pipe_s, d2h = e2e_pipelined(ex, host, device, args.steps, args.warmup, barrier)
        if world > 1:
            t = torch.tensor([seq_s, pipe_s], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            seq_s, pipe_s = t.tolist()
        e2e = {"value": w.total_tokens / pipe_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": pipe_s * 1e3,
               "mode": "pipelined: step i+1's H2D and step i's D2H overlap compute on copy "
                       "streams (double-buffered inputs); host wall clock over all steps",
               "sequential_ms_per_step": seq_s * 1e3}

    # isolated exchange bandwidth (N > 1): min over ranks of the per-rank receive GB/s
    xbw = ex.exchange_benchmark() if world > 1 else None
    if xbw:
        xbw["fwd_transport"] = ("K5 pull kernel (SM loads over NVLink)" if ex.sm_pull
                                else "copy-engine 2-D pulls")
    if xbw is not None:
        for key in ("fwd_kv_pull", "bwd_dkv_return"):
            g = torch.tensor([xbw[key]["GBps"] or 0.0], device=device)
            dist.all_reduce(g, op=dist.ReduceOp.MIN)
            xbw[key]["GBps_min_over_ranks"] = g.item()

    # transparent reshuffler (§8f, N > 1): user layout -> FCP layout for Q/K/V/dO and back
    # for O/LSE/dQ/dK/dV, measured on the comm path, beside the reference's analytic cost
    reshuffle = None
    if world > 1:
        from paper_2605_08524_b200.costmodel import B200_HARDWARE, DEFAULT_EFFICIENCY as _EFF
        from paper_2605_08524_b200.reshuffle import Reshuffler
        from paper_2605_08524_b200.simmodel import default_contiguous_layout, reshuffle_cost
        rs = Reshuffler(result, rank, cfg, device)
        tu = rs.plan.user_tokens
        usr = [torch.randn((tu,) + tuple(x.shape[1:]), device=device).to(x.dtype) for x in (q, k, v, do)]
        fin = ex.step(q, k, v, do)
        tms = []
        for _ in range(4):
            barrier()
            torch.cuda.synchronize()
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(stream)
            rs.to_fcp(*usr)
            b.record(stream)
            rs.from_fcp(*fin)
            c.record(stream)
            torch.cuda.synchronize()
            tms.append((a.elapsed_time(b), b.elapsed_time(c)))
        to_ms, from_ms = sorted(tms)[len(tms) // 2]
        # measured hiding of the to-FCP reshuffle behind the PRE_WAVE tiles (rows that stay
        # on their rank): sequential (reshuffle Q/K/V, then forward) vs forward_user
        ex_u = FcpExecutor(result, rank, cfg, device, resident=rs.resident_chunks())
        # user-layout Q/K/V written where the reshuffler publishes them (no publish copy)
        usr_qkv = rs.input_views([(tuple(x.shape[1:]), x.dtype) for x in usr[:3]])
        for dst_, src_ in zip(usr_qkv, usr[:3]):
            dst_.copy_(src_)
        pre_pairs = sum(wv.pairs for wv in ex_u.work.fwd.waves if wv.stage == -2)
        seq_t, ovl_t, to3_t = [], [], []
        for it in range(5):
            for mode in ("to3", "seq", "ovl"):
                barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                if mode == "to3":
                    rs.to_fcp(*usr_qkv)
                elif mode == "seq":
                    qf, kf, vf = rs.to_fcp(*usr_qkv)
                    ex_u.forward(qf, kf, vf)
                else:
                    ex_u.forward_user(rs, *usr_qkv, overlap=True)
                b.record(stream)
                torch.cuda.synchronize()
                if it:
                    {"to3": to3_t, "seq": seq_t, "ovl": ovl_t}[mode].append(a.elapsed_time(b))
        med = lambda xs: sorted(xs)[len(xs) // 2]
        if os.environ.get("FCPB_BENCH_DEBUG"):
            print(json.dumps({"rank": rank, "to3": to3_t, "seq": seq_t, "ovl": ovl_t}), file=sys.stderr, flush=True)
        t = torch.tensor([to_ms, from_ms, med(seq_t), med(ovl_t), med(to3_t)], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rc = reshuffle_cost(default_contiguous_layout(result.units, n), result.assignment, result.units,
                            result.deps, B200_HARDWARE, cfg, _EFF)
        reshuffle = {"to_fcp_ms_max_over_ranks": t[0].item(), "from_fcp_ms_max_over_ranks": t[1].item(),
                     "fwd_after_to_fcp_ms": t[2].item(), "fwd_user_overlapped_ms": t[3].item(),
                     "to_fcp_qkv_ms": t[4].item(),
                     "hidden_fraction_measured": max(0.0, min(1.0, (t[2].item() - t[3].item()) / t[4].item()))
                     if t[4].item() > 0 else None,
                     "pre_wave_pairs_rank0": pre_pairs,
                     "reference_model": {"to_fcp_ms_at_900GBps": rc.time * 1e3,
                                         "hidden_fraction": rc.hidden_fraction,
                                         "total_bytes": rc.total_bytes}}

    t = torch.tensor([ms], device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = t.item()
    fwd_f, bwd_f = ex.flops()
    total_pairs = batch_token_pairs(list(w.lengths), "causal")
    flop_total = 3.5 * cfg.flops_per_token_pair * total_pairs
    loads = worker_loads(result.assignment, result.units, result.deps, cfg)
    exb = ex.exchange_bytes()

    if rank == 0:
        value = w.total_tokens / (ms_max / 1e3)
        mfu = flop_total / (n * peak * ms_max / 1e3)
        reps = min(3, args.steps)
        kms = {key: sum(s.elapsed_time(e) for s, e in evs) / reps for key, evs in lib_launch.items()}
        nl = {key: len(evs) / reps for key, evs in lib_launch.items()}
        # algorithmic FLOPs per kernel (reference costmodel: fwd 4*Hq*D per pair; the
        # backward's 2.5x splits 4 GEMMs dK/dV + 3 GEMMs dQ of the 7 the split executes,
        # so each kernel is credited its share of the 2.5x: dK/dV 2.5*4/7, dQ 2.5*3/7)
        # recompute dQ executes 4 + 3 GEMM-equivalents for the backward's algorithmic 5;
        # with materialised dS (K2c) the two kernels execute exactly 4 + 1
        ds_mode = ex.op.ds_mode
        kfl = ({"fwd": fwd_f, "bwd": bwd_f * 4 / 5, "dq": bwd_f * 1 / 5} if ds_mode else
               {"fwd": fwd_f, "bwd": bwd_f * 4 / 7, "dq": bwd_f * 3 / 7})
        ktf = {key: (kfl[key] / (kms[key] / 1e3) / 1e12 if kms[key] > 0 else 0.0) for key in kms}
        bwd_ms = kms["bwd"] + kms["dq"]
        bwd_tflops = bwd_f / (bwd_ms / 1e3) / 1e12 if bwd_ms > 0 else 0.0
        top = max(kms, key=lambda kk: kms[kk])
        names = {"fwd": "attn_fwd_kernel", "bwd": "attn_bwd_kernel",
                 "dq": "attn_dqg_kernel" if ds_mode else "attn_dq_kernel"}
        # Algorithmic bytes of the dominant kernel per launch set (reference accounting,
        # DESIGN §5): operands read once and results written once, plus the bf16 dS^T tiles
        # the dK/dV kernel stores (and K2c reads) in materialised-dS mode.
        T_r, R_r = ex.layout.tokens, ex.layout.recv_tokens
        H, Hk, D = cfg.q_heads, cfg.kv_heads, cfg.head_dim
        ds_bytes = (ex.op.ds_bytes if ds_mode else 0)
        alg_bytes = {"fwd": T_r * H * D * 2 * 2 + (T_r + R_r) * Hk * D * 2 * 2 + T_r * H * 4,
                     "bwd": T_r * H * D * 2 * 2 + (T_r + R_r) * Hk * D * 2 * 2 * 2 + T_r * H * 8 + ds_bytes,
                     "dq": T_r * H * D * 2 + (T_r + R_r) * Hk * D * 2 + ds_bytes}
        traffic = measured_traffic(names[top])
        per_launch = alg_bytes[top] / max(nl[top], 1)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong" if args.config in ("c2", "c3") else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": workload_config(w, n, args.scheduler),
            "plan": {"efficiency_curve": args.curve, "plan_ms_host": round(plan_ms, 2),
                     "digest": plan_digest(result, cfg)},
            "mfu": mfu, "flop_total": flop_total,
            # The kernels are timed on their launching stream inside a 3-step pass; the step is
            # tens of ms, so the denominator is the measured burst bf16 peak (the sustained
            # figure applies to seconds-long regions and is shown beside it only).
            "roofline": {"bound": "tensor", "kernel": names[top],
                         "achieved": ktf[top], "peak": peak / 1e12, "unit": "TFLOP/s",
                         "frac": ktf[top] * 1e12 / peak, "peak_kind": peak_kind + " burst (MEASURED_PEAKS.json bf16_tflops)",
                         "peak_sustained": peak_sus / 1e12 if peak_sus else None,
                         "traffic": (traffic["bytes_per_launch"] if traffic else None),
                         "traffic_source": (traffic["source"] if traffic else None),
                         "algorithmic_bytes": per_launch,
                         "traffic_over_algorithmic": (traffic["bytes_per_launch"] / per_launch
                                                      if traffic and per_launch else None),
                         "per_unit": "4*Hq*D FLOP per visible (q,kv) pair (fwd); bwd 2.5x split "
                                     "4/5 dK/dV, 1/5 dQ GEMM (materialised dS) or 4/7, 3/7 "
                                     "(recompute dQ); units = rank-0 visible pairs"},
            "ds_mode": ds_mode,
            "kernels": {names[key]: {"ms": kms[key], "tflops": ktf[key], "frac": ktf[key] * 1e12 / peak,
                                     "launches": nl[key], "algorithmic_bytes": alg_bytes[key]}
                        for key in kms},
            "bwd_total": {"ms": bwd_ms, "tflops": bwd_tflops, "frac": bwd_tflops * 1e12 / peak},
            "exchange_bytes_rank0": exb,
            "exchange_bw_rank0": xbw,
            "reshuffle": reshuffle,
            "phases_ms_rank0": {kk: round(vv, 3) for kk, vv in phases.items()},
            "phases_ms_all_ranks": phases_all,
            "comp_imbalance": (max(loads.compute_flops) - sum(loads.compute_flops) / n) / max(loads.compute_flops),
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "energy": energy,
            "e2e": e2e,
        }
        if not args.no_cpu and n == 1:
            vals, info = cpu_sample(w, result, reps=args.cpu_reps)
            cv = sorted(vals)[len(vals) // 2]
            line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": info["cores"], "kind": "port",
                                    "cpu_model": info["cpu_model"], "sample": info["sample"],
                                    "spread": [min(vals), max(vals)]}
            line["reference_control_plane"] = dict(reference_control_plane(w, n),
                                                   ours_ms=round(plan_ms, 2),
                                                   ours_digest=line["plan"]["digest"])
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
