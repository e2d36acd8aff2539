#!/usr/bin/env python
"""Benchmark: DWM conv2d forward on B200 (images/s, direct-equivalent TFLOP/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                    [--algo auto|exact|tc] [--impl b200|reference]

One step = one full DWM conv2d forward (filter transform, input transform,
transform-domain contraction with the fused output transform) over one
batch of the workload (BASELINE.json configs; default configs[1], the
ResNet-50 stem 7x7/s2 3->64 224x224 batch 256).  Multi-GPU: one process per
GPU (torchrun), every rank runs the full per-GPU batch (weak scaling; images
are independent so there is no collective on the forward path), timed on the
device with CUDA events, max over ranks.

``--impl reference`` times the reference's CPU algorithm (the NumPy port in
oracle/, bit-identical to the reference in the build container) on this
host's cores on a bounded slice of the same workload.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASELINE_METRIC = "DWM conv2d images/s & equiv TFLOP/s at 1/2/4/8 B200; MSE vs FP64 direct conv"
L2_BYTES = 126 * 2 ** 20
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def parse():
    from paper_2002_00552_b200.configs import DEFAULT_WORKLOAD, WORKLOADS
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--algo", default="auto", choices=["auto", "exact", "tc", "small_c"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=None, help="override per-GPU batch (debug only)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank runs the workload's batch; strong: the batch is sharded over ranks")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        out = {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
               "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
               "source": "measured (MEASURED_PEAKS.json)"}
    else:
        out = dict(FALLBACK_PEAKS, bf16_tflops_sustained=1400.0, source="fallback (B200_PROFILING.md)")
    # TF32 tensor and FP32 FFMA peaks measured on this pool's B200s by our own
    # microbenchmarks (tools/tc_probe.cu, tools/fp32_peak.cu); MEASURED_PEAKS has bf16 only
    u = ROOT / "profiles" / "measured_unit_peaks.json"
    if u.exists():
        d = json.loads(u.read_text())
        out["tf32_tflops"], out["fp32_tflops"] = float(d["tf32_tflops"]), float(d["fp32_ffma_tflops"])
        out["unit_source"] = "measured (profiles/measured_unit_peaks.json)"
    else:
        out["tf32_tflops"], out["fp32_tflops"] = out["bf16_tflops"] / 2, 72.0
        out["unit_source"] = "bf16/2 and nominal FP32"
    return out


def small_c_fp32_ops(desc) -> float:
    """FP32 lane operations of the exact-order fused small-C kernel per step:
    per (tile, filter) and part, C*a_r*a_c FMA/MUL (counted as 2 flops), the
    At row/column stage adds and the part-sum adds (SURVEY §8d accounting)."""
    at_nnz = {1: [1, 1], 2: [2, 2], 3: [3, 3]}  # nonzeros per At row
    ops = 0.0
    first = True
    for rp in desc.axis("row"):
        for cp in desc.axis("col"):
            pr, pc = rp[2], cp[2]
            ops += 2.0 * desc.c * (pr + 1) * (pc + 1)
            ops += (pc + 1) * sum(n - 1 for n in at_nnz[pr])
            ops += 2 * sum(n - 1 for n in at_nnz[pc])
            ops += 0 if first else 4
            first = False
    return ops * desc.tiles * desc.f


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.first = threading.Event()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())
            self.first.set()

    def wait_first(self, timeout=5.0):
        if self.proc is not None:
            self.first.wait(timeout)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU arms (oracle = NumPy port of the reference, bit-identical in the build
# container); only used as the reported baseline / the reference arm.
# ---------------------------------------------------------------------------
def cpu_reference_rate(wl, seconds: float, images_per_rep: int = 2, min_reps: int = 2):
    from oracle.dwm_oracle import dwm_conv2d_oracle
    rng = np.random.default_rng(0)
    x = rng.standard_normal((images_per_rep, wl.c_in, wl.hw, wl.hw)).astype(np.float32)
    w = rng.standard_normal((wl.c_out, wl.c_in, wl.kernel, wl.kernel)).astype(np.float32)
    spec = wl.spec()
    dwm_conv2d_oracle(x, w, spec)  # warm (BLAS threads, page-in)
    reps, t0 = 0, time.perf_counter()
    while reps < min_reps or time.perf_counter() - t0 < seconds:
        dwm_conv2d_oracle(x, w, spec)
        reps += 1
    dt = time.perf_counter() - t0
    return images_per_rep * reps / dt, reps, dt


def cpu_threads():
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(var):
            return int(os.environ[var])
    return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args, wl, rank):
    if rank != 0:
        return
    from oracle.dwm_oracle import dwm_conv2d_oracle
    images = 2
    rng = np.random.default_rng(0)
    x = rng.standard_normal((images, wl.c_in, wl.hw, wl.hw)).astype(np.float32)
    w = rng.standard_normal((wl.c_out, wl.c_in, wl.kernel, wl.kernel)).astype(np.float32)
    spec = wl.spec()
    for _ in range(args.warmup):
        dwm_conv2d_oracle(x, w, spec)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        dwm_conv2d_oracle(x, w, spec)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = images * args.steps / total
    cores = cpu_threads()
    sample = (f"{images} images of {wl.name} per step (the reference's NumPy DWM algorithm, "
              f"oracle/dwm_oracle.py port, OpenBLAS {cores} threads, {cpu_model()})")
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": value, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1)",
        "config": {"workload": wl.name, "kernel": wl.kernel, "stride": wl.stride, "pad": wl.pad,
                   "hw": wl.hw, "c_in": wl.c_in, "c_out": wl.c_out, "batch_per_step": images},
        "equiv_tflops": value * wl.direct_flops_per_image() / 1e12,
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    from paper_2002_00552_b200.configs import WORKLOADS
    wl = WORKLOADS[args.workload]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend=backend)

    if args.impl == "reference":
        run_reference_arm(args, wl, rank)
        if dist is not None:
            dist.destroy_process_group()
        return

    from paper_2002_00552_b200 import _native, dwm_conv2d
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    lib = _native.load()
    from paper_2002_00552_b200.sharding import max_over_ranks, shard_range
    global_batch = args.batch or wl.batch
    if args.scaling == "strong":
        lo, hi = shard_range(global_batch, rank, world)
        batch = hi - lo
    else:
        batch = global_batch
    spec = wl.spec()
    desc = _native.make_desc(batch, wl.c_in, wl.hw, wl.hw, wl.c_out, spec.kernel, spec.stride, spec.pad)
    algo = _native.ALGOS[args.algo]
    sel = lib.dwm_select_algo(desc, _native.DWM_F32, algo)
    algo_name = _native.ALGO_NAMES.get(sel, "?")
    ws_bytes = lib.dwm_workspace_bytes(desc, _native.DWM_F32, algo)

    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(batch, wl.c_in, wl.hw, wl.hw, device=dev, generator=gen)
    w = torch.randn(wl.c_out, wl.c_in, wl.kernel, wl.kernel, device=dev, generator=gen)
    y = torch.empty(batch, wl.c_out, desc.oh, desc.ow, device=dev)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    x_bytes, w_bytes, y_bytes = x.numel() * 4, w.numel() * 4, y.numel() * 4
    v_bytes = 0 if algo_name == "small_c" else desc.num_freqs * desc.tiles * wl.c_in * 4
    u_bytes = desc.num_freqs * wl.c_out * wl.c_in * 4 * (2 if algo_name == "tc" else 1)
    working_set = x_bytes + y_bytes + v_bytes
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if working_set < 4 * L2_BYTES else None

    def step():
        st = lib.dwm_conv2d_forward(desc, _native.DWM_F32, algo, x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                    ws.data_ptr(), ws_bytes, flag.data_ptr(), sptr)
        if st:
            _native.check(st, "dwm_conv2d_forward")

    clocks = ClockSampler(dev.index).__enter__()
    clocks.wait_first()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if int(flag.item()):
        raise FloatingPointError("dwm_conv2d produced non-finite values")

    # ---- timed region: K steps, per-step CUDA events on the launching stream
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    n_before = len(clocks.lines)
    if True:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    time.sleep(0.06)
    clocks.__exit__(None, None, None)
    # samples from the warm-up on; keep the timed-region ones when there are enough
    if len(clocks.lines) - n_before >= 3:
        clocks.lines = clocks.lines[n_before:]
    if dist is not None:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = max_over_ranks(sum(step_ms), dist, dev)
    images = (global_batch if args.scaling == "strong" else batch * world) * args.steps
    value = images / (total_ms / 1e3)
    launches_per_step = 2 if algo_name == "small_c" else 3

    # ---- per-stage kernel times (same stream, CUDA events, after the timed region)
    stage_ms = stage_times(lib, desc, algo, algo_name, x, w, y, ws, flag, sptr, stream, flush, reps=max(3, args.steps))

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, wl, spec, batch, dev, dist, world, dwm_conv2d)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    roofline, kernels = make_roofline(stage_ms, desc, wl, batch, algo_name, peaks,
                                      x_bytes, w_bytes, y_bytes, v_bytes, u_bytes)
    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": "images/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1) (torch.randn on device)",
        "config": {"workload": wl.name, "kernel": wl.kernel, "stride": wl.stride, "pad": wl.pad,
                   "hw": wl.hw, "c_in": wl.c_in, "c_out": wl.c_out, "batch_per_gpu": batch,
                   "global_batch": global_batch if args.scaling == "strong" else batch * world,
                   "out_hw": [desc.oh, desc.ow],
                   "parts": desc.n_row_parts * desc.n_col_parts, "frequencies": desc.num_freqs,
                   "engine": algo_name,
                   "l2": ("inputs+intermediates > L2 (%.2f GB/step)" % (working_set / 1e9)
                          if flush is None else "L2 flushed between timed steps (256 MB write)"),
                   "parallelism": f"batch-sharded x{world}, no forward collective"},
        "equiv_tflops": value * wl.direct_flops_per_image() / 1e12,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks.summary(),
        "roofline": roofline,
        "kernels": kernels,
        "e2e": e2e,
    }
    if not args.no_cpu_baseline and world == 1:
        rate, reps, dt = cpu_reference_rate(wl, args.cpu_seconds)
        line["cpu_baseline"] = {
            "value": rate, "unit": "images/s", "cores": cpu_threads(), "kind": "port",
            "sample": (f"{2 * reps} images of {wl.name} in {dt:.1f}s: reference NumPy DWM algorithm "
                       f"(oracle/dwm_oracle.py, bit-identical port), OpenBLAS threads, {cpu_model()}")}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def stage_times(lib, desc, algo, algo_name, x, w, y, ws, flag, sptr, stream, flush, reps):
    """Median CUDA-event time of each kernel the forward launches, run alone."""
    import torch
    from paper_2002_00552_b200 import _native
    ws_ptr = ws.data_ptr()
    v_bytes = 0 if algo_name == "small_c" else desc.num_freqs * desc.tiles * desc.c * 4
    V = ws_ptr
    U = ws_ptr + ((v_bytes + 255) // 256) * 256
    F32 = _native.DWM_F32

    def filt():
        _native.check(lib.dwm_filter_transform(desc, F32, w.data_ptr(), U, sptr))

    def inp():
        _native.check(lib.dwm_input_transform(desc, F32, x.data_ptr(), V, sptr))

    def gemm():
        _native.check(lib.dwm_gemm_output(desc, F32, algo, V, U, y.data_ptr(), flag.data_ptr(),
                                          None, 0, sptr))

    def small_c():
        _native.check(lib.dwm_conv2d_small_c(desc, x.data_ptr(), U, y.data_ptr(), flag.data_ptr(), sptr))

    # one full forward so V/U hold the engine's (layout-specific) contents
    _native.check(lib.dwm_conv2d_forward(desc, F32, algo, x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                         ws_ptr, ws.numel(), flag.data_ptr(), sptr))
    if algo_name == "small_c":
        names = [("filter_transform", filt), ("conv2d_small_c", small_c)]
    elif algo_name == "tc":
        names = [("input_transform", inp), ("gemm_output", gemm)]
    else:
        names = [("filter_transform", filt), ("input_transform", inp), ("gemm_output", gemm)]
    out = {}
    for name, fn in names:
        ms = []
        for _ in range(reps):
            if flush is not None:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        out[name] = statistics.median(ms)
    return out


def make_roofline(stage_ms, desc, wl, batch, algo_name, peaks, x_bytes, w_bytes, y_bytes, v_bytes, u_bytes):
    hbm = peaks["hbm_gbs"]
    gemm_flops = 2.0 * desc.c * desc.f * desc.tiles * desc.num_freqs
    kernels = []
    alg_bytes = {
        "filter_transform": w_bytes + u_bytes,
        "input_transform": x_bytes + v_bytes,
        "gemm_output": v_bytes + u_bytes + y_bytes,
        "conv2d_small_c": x_bytes + u_bytes + y_bytes,
    }
    for name, ms in stage_ms.items():
        k = {"name": name, "ms": ms, "alg_bytes": alg_bytes[name],
             "achieved_gbs": alg_bytes[name] / (ms * 1e-3) / 1e9}
        if name in ("gemm_output", "conv2d_small_c"):
            k["dwm_gemm_flops"] = gemm_flops
            k["achieved_tflops"] = gemm_flops / (ms * 1e-3) / 1e12
        kernels.append(k)
    total = sum(stage_ms.values())
    for k in kernels:
        k["share"] = k["ms"] / total
    top = max(kernels, key=lambda k: k["ms"])
    traffic = lookup_traffic(wl.name, top["name"], batch)
    if top["name"] == "gemm_output" and algo_name == "tc":
        peak_tf32 = peaks["tf32_tflops"]
        achieved = 3 * gemm_flops / (top["ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": top["name"], "achieved": achieved,
                "peak": peak_tf32, "unit": "TFLOP/s", "frac": achieved / peak_tf32,
                "traffic": traffic,
                "note": "3xTF32 tensor FLOPs (3 x 2*C*F*tiles*freqs) vs dense TF32 tcgen05 peak, "
                        + peaks["unit_source"]}
    else:
        achieved = top["alg_bytes"] / (top["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": top["name"], "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                "note": "algorithmic bytes per launch / CUDA-event time vs " + peaks["source"]}
        if top["name"] == "conv2d_small_c":
            fp = small_c_fp32_ops(desc) / (top["ms"] * 1e-3) / 1e12
            roof["fp32_pipe"] = {"achieved": fp, "peak": peaks["fp32_tflops"], "unit": "TFLOP/s",
                                 "frac": fp / peaks["fp32_tflops"],
                                 "note": "C_in<=4: the binding unit is the FP32 pipe (exact reference "
                                         "rounding order on CUDA cores), " + peaks["unit_source"]}
    return roof, kernels


def lookup_traffic(workload, kernel, batch):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
    this kernel from the committed ncu --set full capture, scaled per image to
    this launch's batch; None when no capture exists for the workload."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        e = json.loads(p.read_text()).get(workload, {}).get(kernel)
    except (ValueError, OSError):
        return None
    if not e:
        return None
    return e["bytes_per_image"] * batch


def run_e2e(args, wl, spec, batch, dev, dist, world, dwm_conv2d):
    """Public-API call with pinned HOST buffers: H2D of x and w, the forward,
    D2H of y and of the non-finite flag, every step."""
    import torch
    xh = torch.randn(batch, wl.c_in, wl.hw, wl.hw).pin_memory()
    wh = torch.randn(wl.c_out, wl.c_in, wl.kernel, wl.kernel).pin_memory()
    oh, ow = spec.out_dims(wl.hw, wl.hw)
    yh = torch.empty(batch, wl.c_out, oh, ow).pin_memory()
    for _ in range(2):
        dwm_conv2d(xh, wh, spec, out=yh)
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 5))
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        dwm_conv2d(xh, wh, spec, out=yh)
    torch.cuda.synchronize()
    from paper_2002_00552_b200.sharding import max_over_ranks
    dt = max_over_ranks(time.perf_counter() - t0, dist, dev)
    return {"value": batch * world * steps / dt, "unit": "images/s",
            "h2d_bytes_per_step": (xh.numel() + wh.numel()) * 4,
            "d2h_bytes_per_step": yh.numel() * 4 + 4, "steps": steps,
            "path": "paper_2002_00552_b200.dwm_conv2d(pinned host tensors, out=pinned host tensor)"}


if __name__ == "__main__":
    main()
