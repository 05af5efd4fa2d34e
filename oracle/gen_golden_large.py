"""Full-size golden fixtures from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE (VERDICT r1 "Next round" item 1).  Runs the reference's
own `amplitude_batch` (proj/src/sampler.cpp:111-120 -> execute_slice,
proj/src/engine.cpp:182-245) one slice at a time on the BASELINE configs'
real circuits and plans, so the tests can compare the device engines with
the reference's per-slice contributions on ALL amplitudes at full size:

  config2   7x7 (1+32+1), x1 draw 0, slices 0 and 1 (1024 amplitudes each;
            peak ~52 GB, ~10-20 min per slice on 8 cores)
  config3s  6x10 (1+32+1) stand-in (closed plan): 2 bitstrings x 2 slices
  config5   7x7 (1+40+1), x1 draw 0, slice 5 (64 amplitudes; peak ~35 GB)
  config4s  7x10 (1+32+1) stand-in: 1 bitstring x 1 slice (peak ~103 GB,
            only on a host with that much RAM)
  bc60/bc70 Bristlecone-60/70 (masked 11x12, committed circuit text): one
            bitstring (idle cells 0) x two slices

config2 / bc70 need ~52 GB: they were generated on the GPU box's host
(GOLDEN_OUT=gpurun_out/golden, scripts/gpu_r2_golden.sh) and copied here.

The GEMM is the shim's OpenBLAS cgemm (oracle/shim/Eigen/Core); the BLAS
thread count only splits m / n blocks, so each output element's k-sum is
the same sequence as with one thread.  Usage (here, where /root/reference
exists; outputs are committed under tests/golden/):

    make -C oracle && python oracle/gen_golden_large.py config3s [config5 ...]
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
import qsim_oracle as O  # noqa: E402
import reflib as R  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")

JOBS = {
    "config2": {"circuit": (7, 7, 32, 0), "plan": "configs/config2_plan.json", "x1_draws": [0], "slices": [0, 1]},
    "config5": {"circuit": (7, 7, 40, 0), "plan": "configs/config5_plan.json", "x1_draws": [0], "slices": [5]},
    "config3s": {"circuit": (6, 10, 32, 0), "plan": "configs/config3_standin_6x10_plan.json",
                 "bitstrings": 2, "slices": [0, 1]},
    "config4s": {"circuit": (7, 10, 32, 0), "plan": "configs/config4_standin_7x10_plan.json",
                 "bitstrings": 1, "slices": [0]},
    # Bristlecone-60 on the masked 11x12 embedding (circuit text committed
    # under tests/golden/; parsed by the reference's own parse_circuit).
    "bc60": {"circuit": (11, 12, 32, 0), "mask": 60, "plan": "configs/config3_bristlecone60_plan.json",
             "bitstrings": 1, "slices": [0, 1]},
    # slices 2 and 6 contribute for this bitstring (0 and 1 vanish exactly:
    # inconsistent cut digits; found with the engine, gpurun_out/bc70_nonzero.json)
    "bc70": {"circuit": (11, 12, 32, 0), "mask": 70, "plan": "configs/config4_bristlecone70_plan.json",
             "bitstrings": 1, "slices": [2, 6]},
}
OUT = os.environ.get("GOLDEN_OUT", GOLD)  # e.g. gpurun_out/golden on a host with more RAM


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def run(name: str, threads: int) -> None:
    job = JOBS[name]
    r, c, m, seed = job["circuit"]
    if "mask" in job:
        with open(os.path.join(GOLD, f"bristlecone{job['mask']}_circuit.txt")) as f:
            text = f.read()
    else:
        text = R.generate_rqc(r, c, m, seed)
    plan_text = open(os.path.join(ROOT, job["plan"])).read()
    plan = json.loads(plan_text)
    n = r * c
    open_q = plan["open_qubits"]
    R.lib().ref_set_blas_threads(threads)
    if "x1_draws" in job:
        x1s = [O.draw_x1(n, open_q, 0, d) for d in job["x1_draws"]]
    else:  # closed plan: full bitstrings (closed qubits = x1), fixed numpy stream
        rng = np.random.default_rng(1905)
        x1s = [[int(b) for b in rng.integers(0, 2, n)] for _ in range(job["bitstrings"])]
        if "mask" in job:  # idle cells (H . H) end in |0>
            used = {int(q) for ln in text.splitlines()[1:] if not ln.startswith("#")
                    for q in ln.split()[2:] if ln.split()[1] != "h"}
            for x in x1s:
                for q in range(n):
                    if q not in used:
                        x[q] = 0
    out = {}
    meta = {"name": name, "circuit": list(job["circuit"]), "plan": job["plan"], "slices": job["slices"],
            "x1": x1s, "blas_threads": threads, "cpu": cpu_model(), "nproc": os.cpu_count(),
            "per_slice_flops": plan["per_slice"]["flops"], "seconds": []}
    for i, x1 in enumerate(x1s):
        per = []
        for s in job["slices"]:
            t0 = time.time()
            bits, amps = R.amplitude_batch(text, plan_text, x1, [s])
            dt = time.time() - t0
            meta["seconds"].append(dt)
            print(f"{name} x1#{i} slice {s}: {len(amps)} amplitudes in {dt:.1f} s", flush=True)
            per.append(amps)
        out[f"per_slice{i}"] = np.stack(per)
        out[f"bits{i}"] = np.frombuffer("".join(bits).encode(), dtype=np.uint8).reshape(len(bits), n)
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"large_{name}.npz"), **out)
    with open(os.path.join(OUT, f"large_{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)


def main() -> None:
    threads = int(os.environ.get("REF_BLAS_THREADS", str(os.cpu_count() or 1)))
    for name in sys.argv[1:] or ["config3s"]:
        run(name, threads)


if __name__ == "__main__":
    main()
