"""Benchmark: LLG cell-updates/s of the Grace hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl own|reference]

One JSON line on rank 0.  A "step" is one full LLG step (H_eff by FFT demag +
local terms, Eq. (3), Euler + renormalise) over the whole grid.  Default
workload: the 3-D slab 1024x1024x32 (BASELINE configs[3], paper Sec. 4
material), synthetic seeded random M (workloads.py), inputs resident in HBM.

* value / ms_per_step: CUDA events on the library's stream around grace_step(K)
  (CUDA-graph replay, the product path), after W warm-up steps; the working set
  (>= 3.7 GB) exceeds the 126 MB L2, so no flush is needed.  A second timed
  region runs the same K steps in libgrace profiling mode (every kernel
  bracketed by its own event pair) for the per-kernel split and the roofline.
* roofline: the dominant kernel's algorithmic bytes per launch /
  its mean event-timed duration, against MEASURED_PEAKS.json hbm_gbs.
* e2e: the same metric through the public C-ABI with host buffers: pinned M in
  -> K x (set_hext, step, mavg out) -> M out, all inside the timed region.
* cpu_baseline: the fp64 oracle (oracle/, as it stands) on host cores on a
  bounded sample of the same workload.
* --impl reference: the oracle is this tier's reference arm (no reference code
  exists); it runs on rank 0 only, on a per-step sample sized so K+W steps take
  about two minutes.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import WORKLOADS, random_m  # noqa: E402

METRIC = "LLG cell-updates/s (ms/step) and HBM GB/s fraction at 1/2/4/8 B200"
UNIT = "cell-updates/s"


# ------------------------------------------------------------------ helpers

def algorithmic_bytes(geo, names):
    """Compulsory HBM bytes per launch of each kernel, unpadded Kx.
    K5 writes H_demag (12 B/cell) and K6 reads it back: the split step moves
    24 B/cell more than SURVEY §8(d)'s design (C2R + LLG in one pass)."""
    nx, ny, nz = geo["nx"], geo["ny"], geo["nz"]
    Py, Kx, Kyh, Kzh = geo["Py"], geo["Kx"], geo["Kyh"], geo["Kzh"]
    N = nx * ny * nz
    x1 = 3 * nz * ny * Kx * 8
    x2 = 3 * nz * Py * Kx * 8
    m = 12 * N
    ks = 6 * Kzh * Kyh * Kx * 4 if geo["Pz"] > 1 else 4 * Kyh * Kx * 4
    b = {"K1": m + x1, "K2f": 2 * x1 + ks, "KP": 2 * x1 + ks, "K2": x1 + x2, "K3": 2 * x2 + ks, "K4": x2 + x1,
         "K5": x1 + m, "K6": 3 * m}
    return {k: b[k] for k in names}


def design_step_bytes(geo):
    """SURVEY §8(d)'s per-step compulsory bytes (349 B/cell at the slab): the
    same FFT stages with the C2R and the LLG update in one pass (x1 + 2m)."""
    nx, ny, nz = geo["nx"], geo["ny"], geo["nz"]
    names = kernel_names(geo)
    ab = algorithmic_bytes(geo, names)
    return sum(ab.values()) - 2 * 12 * nx * ny * nz


STEP_DESC = {"K1": "K1 x-R2C", "K2": "K2 y-FFT (TMA)", "K2f": "K2' y-FFT*N*iFFT",
             "KP": "KP plane-fused y-FFT*z-FFT*N*iFFT*iFFT", "K3": "K3 z-FFT*N*iFFT",
             "K4": "K4 y-iFFT (TMA)", "K5": "K5 x-C2R -> H_demag", "K6": "K6 exch+anis+Zeeman+LLG+Euler stencil"}
KERNEL_NAMES = {4: ["K1", "K2f", "K5", "K6"], 6: ["K1", "K2", "K3", "K4", "K5", "K6"]}


def kernel_names(geo):
    """The step's kernels: four with nz = 1 (K2') or on the thin-film plane path (KP), else six."""
    if geo["kernels"] == 4 and geo["Pz"] > 1:
        return ["K1", "KP", "K5", "K6"]
    return KERNEL_NAMES[geo["kernels"]]


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload, kernel):
    """dram read+write bytes per launch from the committed ncu --set full summary, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(workload, {}).get(kernel)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.proc = None
        self.idx = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self, t_start_skip=4):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"]}
        load = rows[t_start_skip:] or rows
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for _, _, r in load for i in range(4) if r[i].lower().startswith("active")})
        return {"sm_mhz": float(np.median([r[0] for r in load])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(load)}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


# ------------------------------------------------------------------ oracle (CPU) legs

REF_LADDER = [(256, 256, 32), (128, 128, 32), (64, 64, 32), (64, 64, 16), (32, 32, 16), (32, 32, 8)]
REF_EST_S = {(256, 256, 32): 4.6, (128, 128, 32): 1.1, (64, 64, 32): 0.25, (64, 64, 16): 0.12,
             (32, 32, 16): 0.03, (32, 32, 8): 0.015}


def oracle_sim(w, n, workers=None, oct_=None):
    from oracle.demag import DemagFFT
    from oracle.llg import Sim
    from oracle.tensor import tensor_octant

    if oct_ is None:
        oct_ = tensor_octant(*n, *w.d)
    op = DemagFFT(oct_, workers=workers)
    return Sim(random_m(n, w.Ms), op, w.Ms, w.A, w.Ku, w.alpha, w.gamma0, w.d, w.hext)


def cpu_baseline(w, steps=3):
    """The oracle as it stands on this host's cores, on a bounded sample of the
    workload: tensor setup timed separately, then Euler steps with numpy's
    single-thread FFT and with scipy.fft on all cores."""
    from oracle.tensor import tensor_octant

    n = (min(256, w.n[0]), min(256, w.n[1]), w.n[2])
    cells = n[0] * n[1] * n[2]
    ncores = host_cores()
    t = time.perf_counter()
    oct_ = tensor_octant(*n, *w.d)
    t_oct = time.perf_counter() - t
    t = time.perf_counter()
    sim = oracle_sim(w, n, oct_=oct_)
    t_spec = time.perf_counter() - t
    sim.euler_step(w.dt)
    t = time.perf_counter()
    sim.run(steps, w.dt)
    el1 = time.perf_counter() - t
    simk = oracle_sim(w, n, workers=ncores, oct_=oct_)
    simk.euler_step(w.dt)
    t = time.perf_counter()
    simk.run(steps, w.dt)
    elk = time.perf_counter() - t
    return {"value": cells * steps / el1, "unit": UNIT, "cores": 1, "kind": "oracle",
            "value_all_cores": cells * steps / elk, "cores_all": ncores,
            "setup_s": {"tensor_octant": t_oct, "kernel_spectrum": t_spec},
            "sample": f"{n[0]}x{n[1]}x{n[2]} cells of the {w.name} workload (same material, cell, dt), "
                      f"1 warm-up + {steps} timed fp64 oracle Euler steps per mode; value: numpy pocketfft "
                      f"single thread ({el1 / steps:.2f} s/step); value_all_cores: scipy.fft workers={ncores} "
                      f"({elk / steps:.2f} s/step); tensor setup (octant + spectrum) {t_oct + t_spec:.1f} s, "
                      f"not in the per-step values"}


def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    budget = 120.0 / max(1, args.steps + args.warmup)
    n = next((s for s in REF_LADDER if REF_EST_S[s] <= budget and s[2] <= w.n[2]), REF_LADDER[-1])
    n = (min(n[0], w.n[0]), min(n[1], w.n[1]), min(n[2], w.n[2]))
    sim = oracle_sim(w, n)
    sim.run(args.warmup, w.dt)
    t = time.perf_counter()
    sim.run(args.steps, w.dt)
    el = time.perf_counter() - t
    cells = n[0] * n[1] * n[2]
    v = cells * args.steps / el
    sample = (f"{n[0]}x{n[1]}x{n[2]} cells of the {w.name} workload per step (same material, cell, dt), "
              f"fp64 oracle (numpy pocketfft, single thread)")
    emit(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "sample_grid": list(n)},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------ own arm

def run_own(args, w):
    import torch

    import paper_1411_2565_b200 as pb

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pb.load()
    nx, ny, nz = w.n
    N = nx * ny * nz
    # GRACE_FORCE_NCCL: the z-slab NCCL path on a one-rank communicator (exercises
    # the multi-GPU plumbing where only one GPU is available)
    distributed = (world > 1 or bool(os.environ.get("GRACE_FORCE_NCCL"))) and nz % world == 0
    if distributed:  # z-slab partition over NCCL (strong scaling of one global grid)
        from paper_1411_2565_b200.dist import create_context, partition

        g = create_context(w, rank, world, local)
        slab = partition(nx, nz, rank, world)
        Mfull = random_m(w.n, w.Ms)
        Mloc = np.ascontiguousarray(Mfull[:, slab.z_offset:slab.z_offset + slab.nz_local])
        del Mfull
        Nloc = Mloc[0].size
    else:  # one grid per GPU (replicas)
        g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, w.gamma0)
        Mloc = random_m(w.n, w.Ms, seed=14112565 + rank)
        Nloc = N
    stream = torch.cuda.Stream()
    pb.grace_set_stream(g.h, stream.cuda_stream)
    M0 = torch.from_numpy(Mloc.astype(np.float32)).cuda()
    pb.grace_set_m_device(g.h, M0.data_ptr())
    g.set_hext(w.hext)
    geo = g.geometry
    names = kernel_names(geo)
    g.step(args.warmup, w.dt)
    # Timed region 1 (the headline): K steps of the product path, CUDA-graph
    # replay with programmatic dependent launch, CUDA events on the library stream.
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        g.step(args.steps, w.dt)
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        # Timed region 2: the same K steps in libgrace profiling mode (eager
        # launches, a CUDA event pair around every kernel on the library stream)
        # for the per-kernel split and the roofline of the dominant kernel.
        profile = not distributed
        kms, klaunch, ms_prof = [0.0] * len(names), [args.steps] * len(names), None
        if profile:
            pb.grace_set_profiling(g.h, True)
            g.step(2, w.dt)  # profiling warm-up (event pool)
            pb.grace_kernel_times(g.h, reset=True)
            ev0.record(stream)
            g.step(args.steps, w.dt)
            ev1.record(stream)
            torch.cuda.synchronize()
            ms_prof = ev0.elapsed_time(ev1) / args.steps
            kms, klaunch = pb.grace_kernel_times(g.h, reset=True)
            pb.grace_set_profiling(g.h, False)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    # distributed: the ranks together step one grid of N cells; replicas: every rank its own
    value = (N if distributed else world * N) * args.steps / (ms / 1e3)

    # roofline of the dominant kernel
    peak, peak_src = read_peaks()
    ab = algorithmic_bytes(geo, names)
    kern = {}
    for name, t, nl in zip(names, kms, klaunch):
        avg = t / max(nl, 1)
        kern[name] = {"ms_per_launch": avg if profile else None, "bytes_per_launch": ab[name],
                      "GBps": ab[name] / (avg / 1e3) / 1e9 if avg > 0 else None,
                      "share": t / sum(kms) if sum(kms) > 0 else None}
    # dominant kernel: the longest measured launch (profiling mode), else the most bytes
    dom = max(kern, key=lambda k: kern[k]["ms_per_launch"] if profile else kern[k]["bytes_per_launch"])
    ach = kern[dom]["GBps"] if profile else None
    step_bytes = sum(ab.values())  # moved by this build's kernels (373 B/cell at the slab)
    design_bytes = design_step_bytes(geo)  # SURVEY §8(d) (349 B/cell at the slab)
    div = world if distributed else 1  # per GPU per step
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak if ach else None,
                "traffic": ncu_traffic(w.name, dom), "peak_source": peak_src,
                "step_bytes_design": design_bytes, "step_bytes_moved": step_bytes,
                "step_frac": design_bytes / div / (ms_step / 1e3) / 1e9 / peak,
                "step_frac_moved": step_bytes / div / (ms_step / 1e3) / 1e9 / peak,
                "step_frac_note": "step_frac: the compulsory bytes of this step's design (SURVEY 8(d): 349 B/cell "
                                  "at the slab; the KP plane path of thin films: K1 + KP + one C2R+LLG pass) "
                                  "/ ms_step / peak; step_frac_moved: the bytes this build's kernels move "
                                  "(K5/K6 split: +24 B/cell)"}

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        # fp32 host buffers (the device state is fp32): 12 B/cell each way
        Mh = torch.empty(3 * Nloc, dtype=torch.float32, pin_memory=True)
        Mh.copy_(torch.from_numpy(np.ascontiguousarray(Mloc, dtype=np.float32).ravel()))
        Mout = torch.empty(3 * Nloc, dtype=torch.float32, pin_memory=True)
        mh = Mh.numpy()
        mo = Mout.numpy()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pb.grace_set_m_f32(g.h, mh)
        for _ in range(args.steps):
            g.set_hext(w.hext)
            g.step(1, w.dt)
            g.mavg()
        pb.grace_get_m_f32(g.h, mo)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        tms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([tms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tms = float(t.item())
        K = args.steps
        e2e = {"value": (N if distributed else world * N) * K / (tms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": (12 * Nloc + 40 * K) / K, "d2h_bytes_per_step": (12 * Nloc + 32 * K) / K,
               "ms_per_step": tms / K, "host_wall_s": wall,
               "api": "grace_set_m_f32(pinned fp32 M) + K x (grace_set_hext, grace_step(1), grace_mavg -> host) + "
                      "grace_get_m_f32(pinned)"}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if distributed else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": w.name, "grid": list(w.n), "cell_m": list(w.d),
                   "padded": [geo["Px"], geo["Py"], geo["Pz"]], "Ms": w.Ms, "A": w.A, "Ku": w.Ku,
                   "alpha": w.alpha, "dt": w.dt, "gamma0": w.gamma0,
                   "l2": f"inputs larger than L2 ({(pb.grace_device_bytes(g.h)) / 1e9:.2f} GB resident vs 126 MB L2); no flush",
                   "parallelism": "single GPU" if world == 1 else
                   (f"z-slab x{world}: " + ("fused P2P transposes (K1/K4 store into peers over NVLink)"
                                            if os.environ.get("GRACE_P2P") == "1" else
                                            "NCCL send/recv transposes pipelined per component")
                    + " + halo planes (one grid)" if distributed
                    else f"{world} independent replicas (nz not divisible by {world})"),
                   "step": " | ".join(STEP_DESC[k] for k in names),
                   "timing": "timed region 1 (value, ms_per_step): K steps of CUDA-graph replay with programmatic "
                             "dependent launch (the step graphs are instantiated in grace_create, none is captured "
                             "inside the region), CUDA events on the library stream; timed region 2 (kernels, "
                             "roofline): the same K steps in libgrace profiling mode, eager launches with a CUDA "
                             "event pair per kernel",
                   "ms_per_step_profiling_mode": ms_prof},
        "roofline": roofline,
        "kernels": kern,
        "gpu_launches": args.steps * len(names),
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(w)
    g.close()
    if rank == 0:
        emit(json.dumps(out))
    if dist:
        dist.destroy_process_group()


_JSON_OUT = None


def emit(line):
    """The one JSON line, on the real stdout (libraries print to fd 1 too: NCCL's
    version banner would otherwise precede it)."""
    out = _JSON_OUT or sys.stdout
    out.write(line + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # keep fd 1 for the JSON line; everything else written to stdout (Python or C
    # libraries) goes to stderr
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="slab_1024x1024x32", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_own(args, w)


if __name__ == "__main__":
    main()
