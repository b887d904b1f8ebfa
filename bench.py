#!/usr/bin/env python3
"""Benchmark: candidate color pairs evaluated per second on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1] [--impl ours|reference]

One step = one pass of the hot path (colorvibe::batch_search, reference
src/search.cpp:403-456) over one batch of synthetic input: by default
BASELINE.json configs[1], the 756-search sweep on the 256 x 1024 grid
(198,180,864 candidates), evaluated in ONE launch of the fused kernel.

Prints ONE JSON line (rank 0):
  value   -- Gcand/s with inputs resident in HBM (device plan; CUDA events on
             the launching stream around each step, L2 flushed between steps)
  e2e     -- same metric through the C-ABI host call `cvg_search` (host
             arrays in; per-target prep, H2D, kernel, D2H of counts + every
             pair record out), wall-clocked per call
  roofline-- FP32-issue roofline of the fused kernel (SURVEY.md §8(d):
             W = 50 FP32 instructions per candidate) vs the FFMA issue peak
             measured in this run
  cpu_baseline -- the reference's own batch_search (oracle/_ref, built from
             the reference sources) on all host cores, same workload

Multi-GPU (torchrun, one process per GPU): weak scaling -- every rank
evaluates its own full copy of the workload; there is no data-path exchange
(the searches are independent), value = all ranks' candidates / max-over-
ranks device time.  `--impl reference` runs the reference CPU arm on rank 0.
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

W_INSTR = 50  # algorithmic FP32 instructions per candidate
METRIC = "candidate color pairs evaluated/sec"
UNIT = "Gcand/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg1", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


@contextlib.contextmanager
def stdout_to_stderr():
    """Points file descriptor 1 at stderr for the duration (C-level prints too)."""
    sys.stdout.flush()
    saved = os.dup(1)
    try:
        os.dup2(2, 1)
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(name):
    from paper_2507_22901_b200 import workloads as W

    return W.ALL[name]()


def config_dict(wl, n, extra=None):
    d = {"workload": f"{wl.name} (BASELINE.json configs[{wl.name[-1]}])", "searches": wl.n_searches,
         "grid": f"{len(wl.radii)} radii x {len(wl.angles)} angles", "candidates_per_step": wl.candidates,
         "targets": {"cfg3": "16^3 lattice", "cfg4": "3840x2160 Voronoi image, one search per pixel"}.get(
             wl.name, "Table-1 colors"), "output": wl.output,
         "parallelism": f"dp{n} (each rank its own {wl.name}-sized batch, no data-path collective)" if n > 1
         else "single", "l2": "flushed between steps (256 MiB write)"}
    if extra:
        d.update(extra)
    return d


# ---------------------------------------------------------------------------
# clocks under load (pynvml, sampled in a thread)

class ClockSampler:
    def __init__(self, device: int, period: float = 0.01):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:  # noqa: BLE001
            pass
        self.period = period
        self._t = threading.Thread(target=self._run, daemon=True)

    REASONS = {
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80, "applications_clocks_setting": 0x2,
    }

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                break
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------

CPU_SAMPLE_SEARCHES = {"cfg4": 20000, "cfg2": 1}  # bounded CPU samples (full cfg0/1/3)


def cpu_sample(wl):
    """Bounded CPU sample of a workload: the first searches (cfg4: 20,000
    pixels, no color memoization; cfg2: one target on 512 of its 4096 radius
    rows), so the reference arm finishes in seconds."""
    n = CPU_SAMPLE_SEARCHES.get(wl.name)
    if n is None:
        return wl, f"full {wl.name} ({wl.n_searches} searches)"
    sub = wl.shard(0, max(1, wl.n_searches // n)) if wl.n_searches > n else wl
    sub = type(wl)(wl.name, sub.targets[:n], sub.patterns[:n], sub.v_th[:n], sub.r_novib[:n], sub.radii,
                   sub.angles, wl.output, wl.note)
    if wl.name == "cfg2":
        sub.radii = wl.radii[::8]
        return sub, f"cfg2 target 0, every 8th radius row ({sub.candidates} candidates)"
    return sub, f"first {n} pixels of {wl.name} ({sub.candidates} candidates, no color memoization)"


def cpu_reference_arm(wl, steps, warmup, cores=None):
    """The reference's own batch_search (oracle/_ref) once per search, all host
    threads, full workload per step.  Returns (Gcand/s, seconds/step, cores)."""
    from oracle.oracle import Reference

    ref = Reference()
    cores = cores or os.cpu_count() or 1
    for _ in range(warmup):
        ref.search_many(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, workers=cores)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        counts = ref.search_many(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, workers=cores)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    return wl.candidates * steps / total / 1e9, total / steps, cores, int(counts.sum()), ref.path


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    wl, sample = cpu_sample(workload(args.config))
    steps = max(1, min(args.steps, 20))
    warm = max(0, min(args.warmup, 2))
    v, sec, cores, pairs, path = cpu_reference_arm(wl, steps, warm)
    out = {
        "metric": METRIC, "value": round(v, 6), "unit": UNIT, "n_gpus": world, "device": "cpu (host cores)",
        "steps": steps, "warmup": warm,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": config_dict(wl, 1, {"cpu": cpu_model(), "library": os.path.relpath(path, ROOT)}),
        "pairs_per_step": pairs,
        "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{sample}: one reference batch_search call per search per step, "
                                   f"workers={cores}"},
        "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def ncu_traffic(config="cfg1"):
    """DRAM bytes (read + write) per launch of phase1_kernel from one committed
    `ncu --set full` capture (profiles/ncu_summary.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("phase1_dram_bytes_per_launch", {}).get(config)
    except (OSError, ValueError):
        return None


def time_gather(dist, plan, wl, n_pairs, world, stream, reps=5):
    """The multi-GPU exchange step of SURVEY §8(e), timed apart from the
    search (scaling is weak: no collective in the timed step): NCCL
    all_gather of every rank's per-search counts, and (PAIRS) of its packed
    pair records (u32 idx + 6 code bytes, padded to the largest rank).  Device
    events around each collective, max over ranks.  The gathered counts are
    checked against the local ones (every rank ran the same batch)."""
    import torch

    n = wl.n_searches
    counts = torch.empty(n, dtype=torch.int64, device="cuda")
    pairs = wl.output == "pairs"
    idx = torch.empty(max(n_pairs, 1), dtype=torch.int32, device="cuda") if pairs else None
    codes = torch.empty((max(n_pairs, 1), 6), dtype=torch.uint8, device="cuda") if pairs else None
    plan.run(stream.cuda_stream)
    plan.sync()
    plan.copy_outputs(counts.data_ptr(), idx.data_ptr() if pairs else 0, codes.data_ptr() if pairs else 0,
                      n_pairs if pairs else 0, stream.cuda_stream)
    sizes = torch.tensor([n_pairs], dtype=torch.int64, device="cuda")
    out_c = [torch.empty_like(counts) for _ in range(world)]

    def timed(fn):
        ms = []
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        v = torch.tensor([statistics.median(ms)], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    out = {"collective": "NCCL all_gather over NVLink", "counts_bytes_per_rank": 8 * n,
           "counts_all_gather_ms": round(timed(lambda: dist.all_gather(out_c, counts)), 4)}
    assert all(torch.equal(x, counts) for x in out_c), "gathered counts differ between ranks"
    if pairs:
        all_sizes = [torch.empty_like(sizes) for _ in range(world)]
        dist.all_gather(all_sizes, sizes)
        width = int(max(int(x.item()) for x in all_sizes))
        rec = torch.zeros((max(width, 1), 10), dtype=torch.uint8, device="cuda")
        rec[:n_pairs, :4] = idx[:n_pairs].view(torch.uint8).view(-1, 4)
        rec[:n_pairs, 4:] = codes[:n_pairs]
        out_r = [torch.empty_like(rec) for _ in range(world)]

        def pairs_gather():
            dist.all_gather(all_sizes, sizes)
            dist.all_gather(out_r, rec)

        out["pairs_bytes_per_rank"] = 10 * n_pairs
        out["pairs_all_gather_ms"] = round(timed(pairs_gather), 4)
        out["pairs_all_gather_gbs"] = round(10 * n_pairs * world / (out["pairs_all_gather_ms"] * 1e-3) / 1e9, 1)
        assert all(torch.equal(x[:n_pairs], rec[:n_pairs]) for x in out_r)
    return out


def run_ours(args):
    import torch

    import paper_2507_22901_b200 as cv

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:  # under torchrun: NCCL even for one rank
        import torch.distributed as dist

        with stdout_to_stderr():  # NCCL prints its version banner on stdout; the JSON line must stand alone
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()  # communicator is created here: keep its banner off stdout too
    wl = workload(args.config)
    ctx = cv.Context(local)
    stream = torch.cuda.current_stream()

    # ---------------- device-resident plan: `value` ----------------
    plan = ctx.plan(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, output=wl.output)
    plan.run(stream.cuda_stream)
    n_pairs = plan.sync()
    if wl.output == "pairs":
        plan.reserve(max(n_pairs, 1))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        flush.zero_()
        plan.run(stream.cuda_stream)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()  # L2 flush outside the timed events
            starts[i].record(stream)
            plan.run(stream.cuda_stream)
            ends[i].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    got = plan.sync()
    assert got == n_pairs, (got, n_pairs)
    kms = plan.last_kernel_ms()  # search kernel alone (last step)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = wl.candidates * world * args.steps / (max_ms * 1e-3) / 1e9

    # per-launch kernel time over the timed steps: events inside the plan
    # cover only the search kernel; re-measure a few steps for the roofline
    # ---- CVG_PATH_PRUNED, reported apart (not the headline): whole radius
    # rows decided by a certified FP64 bound, so its candidates/s counts
    # candidates decided, not each one evaluated ----
    pruned = None
    if wl.output in ("pairs", "counts", "first") and rank == 0 and world == 1:
        pp = ctx.plan(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, output=wl.output,
                      path="pruned")
        pp.run(stream.cuda_stream)
        got_p = pp.sync()
        if wl.output == "pairs":
            pp.reserve(max(got_p, 1))
        for _ in range(args.warmup):
            flush.zero_()
            pp.run(stream.cuda_stream)
        torch.cuda.synchronize()
        p_ms = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            pp.run(stream.cuda_stream)
            b.record(stream)
            torch.cuda.synchronize()
            p_ms.append(a.elapsed_time(b))
        assert pp.sync() == got_p and (wl.output != "pairs" or got_p == n_pairs)
        pruned = {"value": round(wl.candidates * args.steps / (sum(p_ms) * 1e-3) / 1e9, 4), "unit": UNIT,
                  "ms_per_step": round(sum(p_ms) / args.steps, 4), "path": "pruned (CVG_PATH_PRUNED)",
                  "note": "same results; radius rows proven empty by a certified FP64 bound are decided "
                          "without per-candidate evaluation, so this counts candidates decided per second"}
        del pp

    kern, phases = [], []
    plan.set_phase_marks(True)  # events between the kernels (off in the timed steps: they block the PDL overlap)
    for _ in range(min(args.steps, 20)):
        flush.zero_()
        plan.run(stream.cuda_stream)
        kern.append(plan.last_kernel_ms())
        phases.append(plan.last_phase_ms())
    kern_ms = statistics.median(kern)
    phase_ms = [statistics.median(p[i] for p in phases) for i in range(3)]

    # ---------------- e2e through the C-ABI host call ----------------
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 20))
    # warm-up: two calls, so that the shape-hinted buffers of the second call
    # (sized from the first call's pair total) are allocated before timing
    for _ in range(2):
        res = ctx.search(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, output=wl.output)
    assert int(res["n_pairs"]) == n_pairs
    h2d = int(res["stats"]["h2d_bytes"])
    d2h = int(res["stats"]["d2h_bytes"])
    del res
    if dist:
        dist.barrier()
    e2e_times, phases = [], []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        r = ctx.search(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, output=wl.output)
        _ = int(r["n_pairs"])
        e2e_times.append(time.perf_counter() - t0)
        phases.append({k: r["stats"][k] for k in ("prep_ms", "h2d_ms", "device_ms", "d2h_ms", "total_ms")})
        del r
    phase_med = {k: round(statistics.median(p[k] for p in phases), 4) for k in phases[0]}
    e2e_s = sum(e2e_times)
    t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    gather = None
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gather = time_gather(dist, plan, wl, n_pairs, world, stream)
    e2e_value = wl.candidates * world * e2e_steps / float(t.item()) / 1e9

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---------------- roofline ----------------
    # algorithmic output bytes: 10 B per pair + 8 B count per search (pairs);
    # count + first pair (8 + 4 + 6 B) per search (first)
    out_bytes = n_pairs * 10 + wl.n_searches * 8 if wl.output == "pairs" else wl.n_searches * 18
    peak_lane, _ = cv.measure_ffma_peak(local)
    # dominant kernel: phase 1 decides every candidate (the W = 50 algorithmic
    # FP32 instructions of SURVEY §8d); the whole 3-kernel step is reported too
    p1_ms = phase_ms[0] if phase_ms[0] > 0 else kern_ms
    achieved = wl.candidates * W_INSTR / (p1_ms * 1e-3) / 1e12
    peak = peak_lane / 1e12
    step_achieved = wl.candidates * W_INSTR / (kern_ms * 1e-3) / 1e12
    roofline = {"bound": "fp32_issue", "kernel": "phase1_kernel", "achieved": round(achieved, 3),
                "peak": round(peak, 3), "unit": "Tinstr/s", "frac": round(achieved / peak, 4) if peak else None,
                "traffic": ncu_traffic(wl.name), "kernel_ms": round(p1_ms, 4),
                "step_kernels_ms": {"phase1": round(phase_ms[0], 4), "scan": round(phase_ms[1], 4),
                                    "emit": round(phase_ms[2], 4), "total": round(kern_ms, 4)},
                "step_frac": round(step_achieved / peak, 4) if peak else None,
                "instr_per_candidate": W_INSTR,
                "peak_source": "FFMA issue microbenchmark measured in this run (cvg_measure_ffma_peak)",
                "hbm": {"bytes_per_launch": out_bytes,
                        "achieved_gbs": round(out_bytes / (kern_ms * 1e-3) / 1e9, 2)}}

    # ---------------- CPU baseline (reference, bounded sample) ----------------
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cwl, sample = cpu_sample(wl)
            v, sec, cores, pairs, _ = cpu_reference_arm(cwl, 2, 1)
            cpu = {"value": round(v, 6), "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"{sample}, mean of 2 steps after 1 warm-up, workers={cores}, {cpu_model()}",
                   "pairs": pairs, "s_per_step": round(sec, 4)}
            if cwl is wl:
                assert pairs == n_pairs, (pairs, n_pairs)
        except FileNotFoundError as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    out = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64repair", "data": "synthetic",
        "config": config_dict(wl, world, {"pairs_per_step": n_pairs}),
        "e2e": {"value": round(e2e_value, 4), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "s_per_step": round(float(t.item()) / e2e_steps, 5), "steps": e2e_steps,
                "api": "cvg_search (C-ABI host call)", "breakdown_ms": phase_med},
        "gpu_launches": plan.launches * args.steps,
        **({"gather": gather} if gather else {}),
        **({"pruned": pruned} if pruned else {}),
        "clocks": clk.summary(),
        "roofline": roofline,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
