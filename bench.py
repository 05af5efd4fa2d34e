#!/usr/bin/env python3
"""Benchmark of the sliced tensor-network amplitude path (BASELINE.json metric:
amplitudes/sec and sustained Eq.(1) Tflop/s, with the roofline fraction, next
to the reference CPU path on the same host).

Default workload (N=1): BASELINE config 5 -- 7x7 grid RQC depth (1+40+1),
reference_plan_7x7 (1024 slices, rank-30 intermediates), the largest config
that fits one GPU.  One "step" = one slice per GPU; the job is the ascending
select_slices list, split into contiguous per-rank blocks, every rank on the
same x1; a 64-amplitude batch needs 6 slices (fidelity 6/1024, the paper's
run).  The per-slice contributions meet in one NCCL all-gather and an
ascending-slice FP64 merge at the end (checked).  Config 2 (1024-amplitude
batches, 2 slices) instead runs whole x1 batches per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1|2|3|4|5]
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

CONFIGS = {
    "1": {"circuit": (4, 4, 16, 0), "plan": "configs/config1_plan.json",
          "workload": "config1: 4x4 RQC depth (1+16+1), greedy plan, 64-amplitude batch per x1 draw; "
                      "x1 batching: the plan widened to open the 10 x1 qubits serves all 1024 draws "
                      "in one contraction (Engine.amplitude_batches)",
          "slices_per_step": None, "x1_batch": 1024},
    "2": {"circuit": (7, 7, 32, 0), "plan": "configs/config2_plan.json",
          "workload": "config2: 7x7 RQC depth (1+32+1), reference 7x7 region order, 1 cut bond "
                      "b_007_003_004 (2 slices), 1024-amplitude batch per x1 draw",
          "slices_per_step": None},
    "3": {"circuit": (11, 12, 32, 0), "mask": 60, "plan": "configs/config3_bristlecone60_plan.json",
          "workload": "config3: Bristlecone-60 (11x12 diamond embedding) depth (1+32+1), clustered column snake, "
                      "10 cut bonds (K = 1024 slices, max rank 28), closed amplitude over the fixed 2^10-slice set "
                      "(all of K: full fidelity); 1 slice per step per GPU",
          "slices_per_step": 1, "slices_per_batch": 1024},
    "4": {"circuit": (11, 12, 32, 0), "mask": 70, "plan": "configs/config4_bristlecone70_plan.json",
          "workload": "config4: Bristlecone-70 (11x12 diamond embedding) depth (1+32+1), clustered column snake, "
                      "16 cut bonds (K = 65536 slices, max rank 31), closed amplitude over a fixed 2^12-slice "
                      "subset (path fraction 1/16); 1 slice per step per GPU",
          "slices_per_step": 1, "slices_per_batch": 4096},
    "3s": {"circuit": (6, 10, 32, 0), "plan": "configs/config3_standin_6x10_plan.json",
           "workload": "config3 rectangular stand-in: 6x10 RQC depth (1+32+1), column sweep, 12-bond seam cut "
                       "(4096 slices), closed amplitude over a fixed 2^10-slice subset; 1 slice per step per GPU",
           "slices_per_step": 1, "slices_per_batch": 1024},
    "4s": {"circuit": (7, 10, 32, 0), "plan": "configs/config4_standin_7x10_plan.json",
           "workload": "config4 rectangular stand-in: 7x10 RQC depth (1+32+1), column sweep, 12-bond seam cut "
                       "(4096 slices), closed amplitude over a fixed 2^12-slice subset; 1 slice per step per GPU",
           "slices_per_step": 1, "slices_per_batch": 4096},
    "5": {"circuit": (7, 7, 40, 0), "plan": "configs/config5_plan.json",
          "workload": "config5: 7x7 RQC depth (1+40+1), reference_plan_7x7 (1024 slices), 64-amplitude batch at "
                      "fidelity 6/1024 (6 slices per batch, as the paper's run); 1 slice per step per GPU",
          "slices_per_step": 1, "slices_per_batch": 6},
}


def circuit_text(cfg, gen):
    """The config's circuit: generate_rqc (gen = the product's or the
    reference's generator), or for the Bristlecone configs the masked 11x12
    embedding committed as text (tests/golden/bristlecone{60,70}_circuit.txt,
    written by generate_rqc_masked; the reference has no masked generator)."""
    r, c, m, s = cfg["circuit"]
    if "mask" in cfg:
        with open(os.path.join(ROOT, "tests", "golden", f"bristlecone{cfg['mask']}_circuit.txt")) as f:
            return f.read()
    return gen(r, c, m, s)


def idle_qubits(cfg):
    """Cells outside the Bristlecone mask: H . H = identity, so their output bit must be 0."""
    if "mask" not in cfg:
        return []
    text = circuit_text(cfg, None)
    used = set()
    for ln in text.splitlines()[1:]:
        f = ln.split()
        if len(f) >= 3 and not ln.startswith("#") and f[1] != "h":
            used.update(int(x) for x in f[2:])
    return [q for q in range(int(text.split()[0])) if q not in used]


def tc_split(step):
    """Operand split the tcgen05 path uses for a GEMM step (mirrors use_f16 /
    use_3m in csrc/device/cgemm_tc.cu): 3xFP16 on the CTA-pair kernel when
    2k % 64 == 0, as 3M (three real products) when n, k >= 4096."""
    if os.environ.get("QSG_TC_PREC") == "tf32":
        return "3xTF32"
    n2 = 2 * step["n"]
    pair = step["m"] % 256 == 0 and any(n2 % bn == 0 for bn in (256, 128, 64, 32))
    if not (pair and (2 * step["k"]) % 32 == 0):
        return "3xTF32"
    if os.environ.get("QSG_TC_3M", "1") != "0" and step["n"] >= 4096 and step["k"] >= 4096 and step["k"] % 64 == 0:
        return "3M-3xFP16"
    return "3xFP16"


def tc_ceiling(split, bf16):
    """Eq.(1)-equivalent ceiling of a tensor-core GEMM path from the bf16 dense
    rate (f16 = bf16 rate): per complex MAC (8 Eq.1 flop) the 2x2 embedding
    runs 4 real MACs x 3 passes, 3M 3 real MACs x 3 passes, 3xTF32 the
    embedding at half rate."""
    return {"3xFP16": bf16 / 3.0, "3M-3xFP16": bf16 * 4.0 / 9.0, "3xTF32": bf16 / 6.0}[split]


def measured_traffic(kernel_name, class_key=None):
    """DRAM bytes of the dominant kernel from a committed ncu --set full
    capture: profiles/r2_traffic.json by class key ("<split> n=<n> k=<k>"),
    else profiles/r1_traffic.json by the exact step name."""
    for fname, key in (("r2_traffic.json", class_key), ("r1_traffic.json", kernel_name)):
        p = os.path.join(ROOT, "profiles", fname)
        if key is None or not os.path.exists(p):
            continue
        with open(p) as f:
            hit = json.load(f)["kernels"].get(key)
        if hit is not None:
            return hit
    return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, \
        "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                if len(f) >= 7:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[3 + i]
                          and "Not" not in s[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- reference arm

def cpu_reference_sample(cfg, steps_prefix: int, threads: int, seed: int = 0, ntasks: int = 0):
    """Times the reference's own step kernels (oracle/_ref = unmodified qsim
    library, Eigen GEMM -> OpenBLAS 1-thread shim) over the first
    `steps_prefix` plan steps of `ntasks` (default: `threads`) independent
    (x1, slice) tasks on `threads` host threads.  Returns (seconds, flops)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import reflib  # the reference's own generator: nothing from libqsg.so on this arm
    text = circuit_text(cfg, reflib.generate_rqc)
    plan = open(os.path.join(ROOT, cfg["plan"])).read()
    open_q = json.loads(plan)["open_qubits"]
    return reflib.execute_prefix(text, plan, open_q, steps_prefix, ntasks or threads, threads, seed)


def reference_tasks(plan_json: dict, nsteps: int, threads: int, budget_flops: float) -> int:
    """Independent tasks per sample: one per thread, more for small plans so
    the sample is ~budget_flops of CPU work (about 10-30 s)."""
    prefix = sum(st["flops"] for st in plan_json["steps"][:nsteps]) or 1
    return max(threads, min(1 << 20, int(budget_flops // prefix)))


def step_mnk(st: dict):
    """(m, n, k) of a plan step from its annotation: flops = 8 sqrt(vl vr vo),
    intensity = flops / (8 (vl + vr + vo)), volume = vo."""
    import math
    f8 = st["flops"] / 8.0
    vo = float(st["volume"])
    s = st["flops"] / (8.0 * st["intensity"]) - vo  # vl + vr
    p = f8 * f8 / vo                                # vl * vr
    d = math.sqrt(max(s * s - 4 * p, 0.0))
    vl, vr = (s + d) / 2, (s - d) / 2
    k = math.sqrt(vl * vr / vo)
    return int(round(vl / k)), int(round(vr / k)), int(round(k))


def cpu_heavy_gemm_rate(plan_json: dict, threads: int, reps: int = 4):
    """Eq.(1) rate of the reference's contract_ttgt + normalize_inplace on the
    heavy step class (steps >= 1% of a slice's flops), measured on a
    scaled-down copy of the largest step (m, k cut to <= 1024 / 4096; n <=
    4096) run concurrently on `threads` host threads.  Returns (rate, desc)."""
    import threading as th
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import reflib
    top = max(plan_json["steps"], key=lambda x: x["flops"])
    m, n, k = step_mnk(top)
    m, n, k = min(m, 1024), min(n, 4096), min(k, 4096)
    rng = np.random.default_rng(0)
    a = (rng.random((m, k)) + 1j * rng.random((m, k))).astype(np.complex64)
    b = (rng.random((k, n)) + 1j * rng.random((k, n))).astype(np.complex64)
    out = {"flops": 0}
    lock = th.Lock()

    def work():
        for _ in range(reps):
            _, _, fl = reflib.contract_step([0, 1], a, 0.0, [1, 2], b, 0.0, [0, 2], True)
            with lock:
                out["flops"] += fl
    ts = [th.Thread(target=work) for _ in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    secs = time.perf_counter() - t0
    rate = out["flops"] / secs
    return rate, (f"heavy steps at {rate / 1e9:.1f} Eq.1 Gflop/s, measured on a {m}x{n}x{k} contract_ttgt "
                  f"(scaled-down s{plan_json['steps'].index(top):03d}) x{threads} threads in {secs:.1f} s")


def heavy_unmeasured(plan_json: dict, nsteps: int) -> float:
    """Flops of the heavy steps (>= 1% of a slice) outside the measured prefix."""
    total = plan_json["per_slice"]["flops"]
    return sum(st["flops"] for st in plan_json["steps"][nsteps:] if st["flops"] >= 0.01 * total)


def cpu_composite_amps(plan_json: dict, cfg, prefix_rate: float, heavy_rate: float, per_step: int,
                       nsteps: int) -> float:
    """Amplitudes/s of the reference on this host: heavy steps beyond the
    measured prefix at the heavy GEMM rate, everything else at the measured
    plan-prefix rate."""
    total = plan_json["per_slice"]["flops"]
    heavy = heavy_unmeasured(plan_json, nsteps)
    secs_per_slice = heavy / heavy_rate + (total - heavy) / prefix_rate
    slices = cfg.get("slices_per_batch") or per_step
    return (1 << len(plan_json["open_qubits"])) / (secs_per_slice * slices)


def reference_prefix_steps(plan_json: dict, budget_flops: float) -> int:
    """Longest plan prefix whose Eq.(1) flops stay within budget_flops (>= 1 step)."""
    acc, n = 0, 0
    for st in plan_json["steps"]:
        if acc + st["flops"] > budget_flops and n > 0:
            break
        acc += st["flops"]
        n += 1
    return n


def host_cpu():
    """(nproc, CPU model) of this host, reported next to every CPU number."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def reference_anchor():
    """The composite model checked against one COMPLETE stock reference
    slice (scripts/ref_anchor.py -> profiles/ref_anchor.json), if recorded."""
    p = os.path.join(ROOT, "profiles", "ref_anchor.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return {k: d[k] for k in ("config", "measured_s", "model_s", "measured_over_model", "host", "note") if k in d}


def cpu_baseline_record(value, threads, sample):
    nproc, model = host_cpu()
    rec = {"value": value, "unit": "amplitudes/s", "cores": threads, "kind": "reference", "extrapolated": True,
           "nproc": nproc, "cpu_model": model, "sample": sample}
    anchor = reference_anchor()
    if anchor:
        rec["anchor"] = anchor
    return rec


def run_reference_arm(args):
    world, rank, local = dist_setup()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    plan = json.load(open(os.path.join(ROOT, cfg["plan"])))
    nproc = os.cpu_count() or 1
    threads = args.cpu_threads or min(nproc, 32)
    nsteps = reference_prefix_steps(plan, args.cpu_budget_flops)
    prefix_flops = sum(s["flops"] for s in plan["steps"][:nsteps])
    batch = 1 << len(plan["open_qubits"])
    slices_per_batch = cfg.get("slices_per_batch") or plan["slices"]
    flops_per_step = plan["per_slice"]["flops"] * slices_per_batch
    ntasks = reference_tasks(plan, nsteps, threads, args.cpu_budget_flops / 4)
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, nsteps, threads, ntasks=threads)
    secs, flops = 0.0, 0
    for i in range(args.steps):
        s, f = cpu_reference_sample(cfg, nsteps, threads, seed=i + 1, ntasks=ntasks)
        secs += s
        flops += f
    rate = flops / secs  # Eq.(1) flop/s of the reference kernels on this host (plan prefix)
    heavy_rate, heavy_desc = (cpu_heavy_gemm_rate(plan, threads) if heavy_unmeasured(plan, nsteps) > 0
                              else (rate, "no heavy steps beyond the prefix"))
    amps = cpu_composite_amps(plan, cfg, rate, heavy_rate, slices_per_batch, nsteps)
    rate_eff = amps / batch * flops_per_step
    line = {
        "metric": "amplitudes_per_sec", "value": amps, "unit": "amplitudes/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c64 (fp32)",
        "data": "synthetic (seeded RQC, random x1)",
        "config": {"workload": cfg["workload"], "parallelism": f"{threads} host threads"},
        "tflops_eq1": rate_eff / 1e12,
        "cpu_baseline": cpu_baseline_record(
            amps, threads,
            f"EXTRAPOLATED: reference qsim kernels (contract_ttgt + normalize_inplace, Eigen GEMM via "
            f"OpenBLAS 1-thread shim) over plan steps s000..s{nsteps - 1:03d} "
            f"({prefix_flops / plan['per_slice']['flops']:.2%} of a slice's Eq.1 flops) of "
            f"{ntasks} independent (x1, slice) tasks per step on {threads} threads at "
            f"{rate / 1e9:.1f} Eq.1 Gflop/s; {heavy_desc}; amplitudes/s = batch / "
            f"(heavy flops / heavy rate + other flops / prefix rate); ms_per_step is the timed sample, "
            f"not a batch"),
        "e2e": {"value": amps, "unit": "amplitudes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ----------------------------------------------------------------------------- our arm

def run_ours(args):
    import numpy as np
    import torch

    import paper_1905_00444_b200 as Q

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    r, c, m, s = cfg["circuit"]
    text = circuit_text(cfg, Q.generate_rqc)
    idle = idle_qubits(cfg)
    plan_text = open(os.path.join(ROOT, cfg["plan"])).read()
    plan = json.loads(plan_text)
    rewrites = None
    if args.reassociate:
        plan_text, rewrites = Q.reassociate_plan(text, plan_text)
    open_q = plan["open_qubits"]
    n = r * c
    xb = args.x1_batch if args.x1_batch is not None else cfg.get("x1_batch", 1)
    closed = [q for q in range(n) if q not in open_q]
    if xb > 1:
        if cfg["slices_per_step"] is not None or len(closed) > 20 or xb > (1 << len(closed)):
            raise SystemExit("--x1-batch needs batch mode, <= 20 x1 qubits and at most 2^#x1 draws")
        eng_plan = Q.widen_plan(text, plan_text, closed)
    else:
        eng_plan = plan_text
    eng = Q.Engine(text, eng_plan, device=local, tensor_cores=not args.no_tc, memory_budget=args.memory_budget)
    info = eng.info
    K = plan["slices"]
    per_step = cfg["slices_per_step"] or K
    batch = xb * (1 << len(open_q))  # amplitudes delivered per run

    from paper_1905_00444_b200 import distributed as D
    slice_mode = cfg["slices_per_step"] is not None
    if slice_mode:
        # One sliced job: the ascending select_slices list of steps x world
        # x per_step slices (src/engine.cpp:285-298), contiguous blocks per
        # rank; every rank contracts the SAME x1 (draw 0).
        njob = min(args.steps * world * per_step, K)
        job_ids = Q.select_slices(njob, K, K, 0)
        blocks = D.slice_blocks(job_ids, world)
        mine = blocks[rank]

    def slices_for(step_index: int):
        """Slices of timed step `step_index` (warm-up steps reuse step 0's)."""
        if not slice_mode:
            return list(range(K))
        i = max(step_index - args.warmup, 0)
        return [mine[(i * per_step + j) % len(mine)] for j in range(per_step)]

    # ---- device-timed region: node tensors resident, slices back to back ----
    def draw(seed, index):
        x = Q.draw_x1(n, open_q, seed, index)
        for q in idle:  # idle Bristlecone cells end in |0>
            x[q] = 0
        return x

    x1 = (draw(0, 0 if slice_mode else rank) if xb == 1 else [-1] * n)
    eng.prepare(x1)
    eng.synchronize()
    for w in range(args.warmup):
        eng.run(slices_for(w), reset=True, per_slice=True)
    eng.synchronize()
    stream = torch.cuda.ExternalStream(eng.stream(), device=local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = eng.launches()
    # Working sets below ~2x L2 (config 1): flush L2 (write 256 MiB) between
    # steps, outside the per-step event windows.
    small = info.arena_bytes < (256 << 20)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if small else None

    def timed_run(i):
        # batch mode: every step is a whole batch (reset); slice mode: the
        # rank's block accumulates across steps, one per-slice row per slice.
        eng.run(slices_for(args.warmup + i), reset=(not slice_mode or i == 0), per_slice=True)

    with ClockSampler(local) as clocks:
        if small:
            ms = 0.0
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            with torch.cuda.stream(stream):
                for i in range(args.steps):
                    flush.fill_(i & 255)
                    evs[i][0].record(stream)
                    timed_run(i)
                    evs[i][1].record(stream)
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs)
        else:
            ev0.record(stream)
            for i in range(args.steps):
                timed_run(i)
            ev1.record(stream)
            ev1.synchronize()
            ms = ev0.elapsed_time(ev1)
    torch.cuda.synchronize()
    launches = eng.launches() - launches0
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    # batch mode: every step is a full amplitude batch; slice mode: a batch
    # needs `slices_per_batch` slices (fidelity fraction / fixed subset).
    amps_total = batch * args.steps * world * per_step / cfg.get("slices_per_batch", per_step)
    flops_total = info.flops_per_slice * per_step * args.steps * world
    value = amps_total / (ms / 1e3)
    tflops = flops_total / (ms / 1e3) / 1e12
    amps_local, rows = eng.results(per_slice=True)

    # ---- the one collective (NCCL over NVLink) and its checks.
    merge = None
    dev_t = torch.device("cuda", local)
    if slice_mode:
        # K3's FP64 accumulator over the rank's block == the ascending sum of
        # its per-slice rows, bit for bit (src/engine.cpp:352-356 order).
        local_ok = bool(np.array_equal(D.ordered_merge(rows), amps_local))
        allc = D.gather_contributions(rows, [len(bk) for bk in blocks], device=dev_t) if world > 1 else rows
        merged = D.ordered_merge(allc)
        cross_ok = None
        if world > 1:
            # per-slice contributions do not depend on the GPU: rank 0
            # recomputes rank 1's first slice and must match its row exactly,
            # so the merged batch equals the single-GPU run bit for bit.
            if rank == 0:
                eng.run([blocks[1][0]], reset=True, per_slice=True)
                _, chk = eng.results(per_slice=True)
                cross_ok = bool(np.array_equal(chk[0], allc[len(blocks[0])]))
            flags = torch.tensor([int(local_ok)], device=dev_t)
            torch.distributed.all_reduce(flags, op=torch.distributed.ReduceOp.MIN)
            local_ok = bool(flags.item())
        if not local_ok or cross_ok is False:
            raise SystemExit(f"sliced merge check failed (local {local_ok}, cross-GPU {cross_ok})")
        merge = {"slices": len(job_ids), "x1_draw": 0, "per_rank_block": len(mine),
                 "checks": "per-rank K3 sum == ordered sum of its per-slice rows (bit-exact)"
                           + ("; rank 0 recomputed rank 1's first slice: bit-identical row" if world > 1 else ""),
                 "amplitude_norm2": float(np.vdot(merged, merged).real)}
        if world > 1:
            merge["collective"] = "1x NCCL all_gather of per-slice FP64 contributions + ascending-slice merge"
    elif world > 1:
        D.gather_contributions(amps_local[None, :], [1] * world, device=dev_t)
        merge = {"collective": "1x NCCL all_gather of the per-rank x1 batches (independent amplitude batches)"}

    # ---- end-to-end through the public API, every step: H2D of the circuit's
    # node tensors (the host open fold, pinned) -> Engine.load_nodes, host x1
    # -> Engine.amplitude_batch(es) (node views, kernels), D2H of the amplitudes.
    h2d = info.node_bytes
    d2h = info.batch_size * 16
    # host inputs of every step (the fold, src/network.cpp:106-155, and the
    # x1 draws, src/sampler.cpp:70-82) are made before the timed region
    host_nodes = torch.empty(info.node_bytes // 8, dtype=torch.complex64, pin_memory=True)
    eng.fold_nodes(text, out=host_nodes)
    host_x1 = [np.asarray([draw(0, 0) if slice_mode else
                           draw(1, (rank * args.steps + i) * xb + t) for t in range(xb)],
                          dtype=np.int32) for i in range(max(args.steps, 2))]
    def e2e_step(i):
        eng.load_nodes(host_nodes)
        if xb == 1:
            eng.amplitude_batch(host_x1[i][0], slices_for(args.warmup + i))
        else:
            eng.amplitude_batches(open_q, host_x1[i], slices_for(args.warmup + i), bitstrings=False)

    def e2e_pipelined(steps):
        # x1 batching (config 1): two batches in flight -- the host gathers
        # batch i from its pinned slot while the GPU runs batch i + 1 (each
        # step still uploads its node tensors and reads its amplitudes back).
        def submit(i):
            eng.load_nodes(host_nodes)
            eng.amplitude_batches_submit(open_q, host_x1[i], slices_for(args.warmup + i), slot=i % 2)
        submit(0)
        for i in range(steps):
            if i + 1 < steps:
                submit(i + 1)
            eng.amplitude_batches_collect(i % 2)

    e2e_step(0)  # untimed warm-up of the API path (pinned staging, graph key)
    if xb > 1:
        e2e_pipelined(2)
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    if xb > 1:
        e2e_pipelined(args.steps)
    else:
        for i in range(args.steps):
            e2e_step(i)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = amps_total / e2e_s

    # ---- roofline: per-op CUDA-event timing on the engine stream (separate pass)
    eng.set_profile(True)
    eng.reset_profile()
    eng.prepare(x1)
    eng.run(slices_for(0), reset=True)
    prof = eng.profile()
    eng.set_profile(False)
    if args.profile_out and rank == 0:
        with open(args.profile_out, "w") as f:
            for p in sorted(prof, key=lambda p: -p["ms_total"]):
                if p["executions"] > 0:
                    f.write(json.dumps(p) + "\n")
    peaks, peak_src = load_peaks()
    gemms = [p for p in prof if p["kind"] == 1 and p["executions"] > 0]
    perms = [p for p in prof if p["kind"] == 0 and p["executions"] > 0]
    total_ms = sum(p["ms_total"] for p in prof)
    # Dominant kernel = the GEMM class (pipe, n, k) with the most time: one
    # launch for the big configs' top step; for the sweep plans (configs 3/4)
    # the ~20 k = n = 256 launches at m = 2^20..2^23.  Per-launch figures are
    # the class averages (sum of flops or bytes / sum of launches).
    classes = {}
    for p in gemms:
        classes.setdefault((p["tensor_cores"], p["n"], p["k"]), []).append(p)
    members = max(classes.values(), key=lambda ps: sum(p["ms_total"] for p in ps))
    execs = sum(p["executions"] for p in members)
    top = dict(max(members, key=lambda p: p["ms_total"]))
    top["ms_total"] = sum(p["ms_total"] for p in members)
    top["flops"] = sum(p["flops"] * p["executions"] for p in members) / execs
    top["bytes"] = sum(p["bytes"] * p["executions"] for p in members) / execs
    top["executions"] = execs
    top_ms = top["ms_total"] / execs
    achieved = top["flops"] / (top_ms / 1e3) / 1e12
    clk = clocks.summary()
    smx = peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * 2 * smx * 1e6 / 1e12
    split = tc_split(top)
    if top["tensor_cores"]:
        how = {"3xFP16": "/ 3 (passes)", "3M-3xFP16": "x 4/9 (3M: 3 real products x 3 passes per 4 MACs)",
               "3xTF32": "/ 2 (tf32) / 3 (passes)"}[split]
        bound, peak_val, peak_note = "tensor", tc_ceiling(split, peaks["bf16_tflops"]), (
            f"{split} ceiling = {peak_src} bf16 dense {peaks['bf16_tflops']} TF/s {how}")
    else:
        bound, peak_val, peak_note = "tensor", fp32_peak, (f"FP32 FFMA peak 148 SM x 128 lanes x 2 x "
                                                           f"{smx:.0f} MHz ({peak_src} sm_max_mhz)")
    if top["bytes"] > 0 and top["flops"] / top["bytes"] < peak_val * 1e12 / (peaks["hbm_gbs"] * 1e9):
        # arithmetic intensity below that ceiling's ridge (e.g. m = 2^28, n = k = 16:
        # 8 flop/B): the step is HBM-bound whatever pipe it runs on
        bound, peak_val, peak_note = "hbm", peaks["hbm_gbs"], (
            f"{peak_src} HBM copy bandwidth (GB/s); algorithmic bytes 8 (mk + kn + mn) of the step")
        achieved = top["bytes"] / (top_ms / 1e3) / 1e9
    simt_name = "cgemm_narrow" if top["n"] <= 32 and top["m"] >= 1024 else "cgemm_simt"
    if len(members) == 1:
        kernel_name = (f"cgemm_tc ({split})" if top["tensor_cores"] else simt_name) + \
            f" step s{top['step']:03d} m={top['m']} n={top['n']} k={top['k']}"
    else:
        ms_ = sorted(p["m"] for p in members)
        kernel_name = (f"cgemm_tc ({split})" if top["tensor_cores"] else simt_name) + \
            f" class n={top['n']} k={top['k']}: {len(members)} steps, m={ms_[0]}..{ms_[-1]} ({execs} launches)"
    perm_ms = sum(p["ms_total"] for p in perms)
    perm_bytes = sum(p["bytes"] * p["executions"] for p in perms)
    roof = {"bound": bound, "achieved": achieved, "peak": peak_val, "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
            "frac": achieved / peak_val,
            "traffic": None, "kernel": kernel_name,
            "kernel_share_of_step": top["ms_total"] / total_ms, "peak_source": peak_note,
            "fp32_simt_peak_tflops": fp32_peak,
            "permute_gbs": (perm_bytes / (perm_ms / 1e3) / 1e9) if perm_ms > 0 else None,
            "permute_share_of_step": perm_ms / total_ms, "hbm_peak_gbs": peaks["hbm_gbs"]}
    traffic = measured_traffic(kernel_name, f"{split} n={top['n']} k={top['k']}" if top["tensor_cores"] else None)
    if traffic is not None:
        roof["traffic"] = traffic["dram_read_bytes"] + traffic["dram_write_bytes"]
        roof["traffic_unit"] = "bytes per launch"
        roof["traffic_source"] = traffic["report"]
        roof["traffic_algorithmic"] = traffic["algorithmic_bytes"]

    tc_share = sum(p["ms_total"] for p in gemms if p["tensor_cores"]) / max(total_ms, 1e-30)
    if tc_share > 0.5:
        dtype_label = (f"c64 (tcgen05 3xFP16 split of fp32 operands, fp32 accumulate{', 3M products on the n, k >= 4096 steps' if any(tc_split(p) == '3M-3xFP16' for p in gemms if p['tensor_cores']) else ''}: "
                       f"{tc_share:.0%} of the step; the rest FP32 FFMA / data movement)")
    else:
        dtype_label = (f"c64 (fp32 FFMA SIMT / narrow GEMMs; tensor cores {tc_share:.0%} of the step)")
    line = None
    if rank == 0:
        line = {
            "metric": "amplitudes_per_sec", "value": value, "unit": "amplitudes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype_label,
            "data": "synthetic (seeded RQC from generate_rqc, random x1 via mt19937_64)",
            "config": {"workload": cfg["workload"], "parallelism": (f"x1 batches across {world} GPU(s)" if cfg["slices_per_step"] is None else f"slices across {world} GPU(s)"),
                       "amplitudes_per_step_per_gpu": batch, "slices_per_step_per_gpu": per_step,
                       **({"x1_draws_per_contraction": xb} if xb > 1 else {}),
                       "flops_per_step_per_gpu": info.flops_per_slice * per_step,
                       "l2": ("working set < 2x L2: 256 MiB L2 flush between steps, outside the per-step "
                              "event windows" if small else
                              f"working set ({info.arena_bytes / 2**30:.1f} GiB arena) >> 126 MB L2; no flush needed"),
                       "arena_bytes": info.arena_bytes, "tensor_cores": not args.no_tc,
                       **({"memory_budget": args.memory_budget} if args.memory_budget else {}),
                       **({"plan": f"reassociated ({rewrites} tree rewrites; Eq.1 flops/slice "
                                   f"{info.flops_per_slice:.4g} vs the plan's {plan['per_slice']['flops']:.4g})"}
                          if rewrites is not None else {})},
            "tflops_eq1": tflops, "tflops_frac_fp32_simt": tflops / fp32_peak,
            "e2e": {"value": e2e_value, "unit": "amplitudes/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "note": "per step: H2D of the circuit's node tensors (host open fold, pinned) + host x1 "
                            "through the Engine API; D2H = batch amplitudes" +
                            ("; x1 batches pipelined two deep (amplitude_batches_submit / _collect)" if xb > 1
                             else "")},
            "gpu_launches": launches, "clocks": clk, "roofline": roof,
        }
        if merge is not None:
            line["config"]["merge"] = merge
    if world > 1:
        torch.distributed.barrier()
    # CPU baseline: rank 0 at N=1 only.
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu_threads = args.cpu_threads or min(os.cpu_count() or 1, 32)
            nsteps = reference_prefix_steps(plan, args.cpu_budget_flops)
            ntasks = reference_tasks(plan, nsteps, cpu_threads, args.cpu_budget_flops / 4)
            secs, fl = cpu_reference_sample(cfg, nsteps, cpu_threads, ntasks=ntasks)
            rate = fl / secs
            heavy_rate, heavy_desc = (cpu_heavy_gemm_rate(plan, cpu_threads) if heavy_unmeasured(plan, nsteps) > 0
                                      else (rate, "no heavy steps beyond the prefix"))
            # the reference runs the plan as given: its flops and batch per x1 draw
            cpu_amps = cpu_composite_amps(plan, cfg, rate, heavy_rate, per_step, nsteps)
            line["cpu_baseline"] = cpu_baseline_record(
                cpu_amps, cpu_threads,
                f"EXTRAPOLATED: unmodified reference kernels (oracle/_ref, Eigen->OpenBLAS 1-thread shim) over "
                f"plan steps s000..s{nsteps - 1:03d} of {ntasks} (x1, slice) tasks on {cpu_threads} "
                f"threads in {secs:.1f} s at {rate / 1e9:.1f} Eq.1 Gflop/s; {heavy_desc}; "
                f"amplitudes/s = batch / (heavy flops / heavy rate + other flops / prefix rate)")
        except Exception as exc:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "unit": "amplitudes/s", "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {exc}"}
    if rank == 0:
        emit(line)
    eng.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


_JSON_FD = 1


def emit(line):
    """The result line goes to the real stdout; everything else (NCCL's
    version banner, library chatter) was redirected to stderr by main()."""
    os.write(_JSON_FD, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="5",
                    help="BASELINE config: 5 (default: the largest single-GPU config), 1, 2, 3/4 (Bristlecone-60/70), "
                         "3s/4s (rectangular stand-ins)")
    ap.add_argument("--no-tc", action="store_true", help="disable the tcgen05 GEMM path")
    ap.add_argument("--reassociate", action="store_true",
                    help="opt-in contraction-tree rewrite of the plan (Q.reassociate_plan); off for the headline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-out", default="", help="write the per-op profile (one JSON line per op) here")
    ap.add_argument("--x1-batch", type=int, default=None,
                    help="x1 draws per contraction via the widened plan (batch-mode configs; config 1 default 1024)")
    ap.add_argument("--memory-budget", type=int, default=0,
                    help="bytes per contraction (reference ExecOptions); larger steps run out of core")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--cpu-budget-flops", type=float, default=4e11,
                    help="Eq.1 flops per task of the reference CPU sample (plan prefix)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
