#!/usr/bin/env python
"""DF11 decompression benchmark (BASELINE.json metric: GB/s of BF16 produced; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama8b_block] [--kernel auto]
    torchrun --nproc-per-node N bench.py --gpus N ...        # one rank per GPU, weak scaling
    python bench.py --impl reference ...                     # the CPU oracle as the reference arm

A step = one df11_decompress_block call over every tensor of one transformer block (all §8(a) rows:
tile map, LUT staging, chunk staging, gaps, phase 1, scan, phase 2, write-back), inputs resident in
HBM.  Each rank decodes its own block (different seeds): no collective on the data path and NCCL is
never initialised; a gloo (CPU) group aligns the start (barrier) and combines the per-rank timings
(max) and byte counts (sum).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "DF11 decompress GB/s (BF16 out) per GPU and 8-GPU aggregate; % of HBM roofline"
UNIT = "GB/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=400)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default=workloads.BASELINE_CONFIGS[1])
    p.add_argument("--kernel", choices=["auto", "alg1", "fast"], default="auto")
    p.add_argument("--format", choices=["256x8", "128x16"], default="256x8",
                   help="DF11 format parameters T x n (P:138: n = 8; 128x16 halves the gap bits, NEXT-4)")
    p.add_argument("--vf", choices=list(workloads.VALUE_FORMATS), default="bf16",
                   help="value format (NEXT-4, P:609): the paper's BF16, or FP16 / FP8 E4M3 / FP8 E5M2 weights of "
                        "the same N(0, 0.02) recipe (value = GB/s of decoded words out)")
    p.add_argument("--lut-bits", default="8",
                   help="b of the format's b-bit LUTs (App. I.2; 8 = the paper) or 'mono' (App. I.1, b = L)")
    p.add_argument("--dist", choices=["gauss", "t5", "sigma-lu"], default="gauss",
                   help="weight distribution: gauss = the headline recipe; t5 / sigma-lu = realism variants")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true",
                   help="skip the extra CUDA-graph replay of the same K steps (reported as 'graph')")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-transfer", action="store_true", help="skip the CPU->GPU transfer baseline (NEXT-2)")
    p.add_argument("--selftest-dist", action="store_true",
                   help="host-side multi-rank check without a GPU: gloo group, per-rank shard placement and "
                        "the whole-job aggregation of synthetic per-rank bytes/times (tests/test_shard_dist.py)")
    p.add_argument("--unique-blocks", type=int, default=2,
                   help="model configs: distinct encoded blocks per rank (device copies fill the shard)")
    return p.parse_args()


# --------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    """Samples SM clock and throttle reasons every 10 ms during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def measured_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def run_env(dev) -> dict:
    """GPU name, driver, torch / CUDA versions and the library build of this run."""
    import torch
    env = {"gpu": torch.cuda.get_device_name(dev), "torch": torch.__version__, "cuda": torch.version.cuda}
    try:
        import pynvml
        pynvml.nvmlInit()
        drv = pynvml.nvmlSystemGetDriverVersion()
        env["driver"] = drv.decode() if isinstance(drv, bytes) else drv
    except Exception:                                                     # reported, never fatal
        pass
    try:
        from paper_2504_11651_b200 import df11
        env["library"] = df11.lib().df11_version().decode()
    except Exception:
        pass
    return env


def variant_key(args) -> str:
    """Suffix of the ncu summary key for a NEXT-4 format variant ("" for the paper's format)."""
    if args.vf == "bf16" and str(args.lut_bits) == "8" and args.format == "256x8":
        return ""
    return f"/{args.vf}-b{args.lut_bits}-{args.format}"


def ncu_traffic(config: str, kernel: str):
    """Per-launch dram bytes from the committed ncu summary (profiles/ncu_summary.json), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(f"{config}/{kernel}")
    return None if e is None else e.get("dram_bytes_per_launch")


# --------------------------------------------------------------------------- CPU oracle timing
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _word_np(vf):
    return np.int16 if workloads.word_dtype(vf) is np.uint16 else np.uint8


def oracle_decode_rate(tensors_np, budget_s: float = 8.0, vf: str = "bf16", lut_bits=8):
    """Time the CPU oracle on a bounded sample of this workload (whole tensors in config order until
    ~budget_s of single-thread work), two ways (SURVEY 8(d) "CPU oracle timing"):
      D1: the sequential decoder, all host cores over the format blocks (started at each block's first
          code, which Gaps / BlockOutputPos locate);
      D2: the Algorithm 1 emulator with all host cores spread over the format blocks of each tensor.
    Returns the cpu_baseline dict (value = the faster of the two, with the threads it used)."""
    import concurrent.futures as cf

    import oracle
    fmts = []
    spent = 0.0
    est_rate = 60e6                                      # el/s per thread (D1), for the sample size
    for name, w in tensors_np:
        if fmts and spent + w.size / est_rate > budget_s:
            break
        fmts.append((name, oracle.encode(w.reshape(-1), vf=vf, lut_bits=lut_bits), w))
        spent += w.size / est_rate
    elems = sum(w.size for _, _, w in fmts)
    host_cores = os.cpu_count() or 1

    # D1: every host core on the format blocks of each tensor (the sequential decoder started at each
    # block's first code: bit 8nT*b + gap, element BlockOutputPos[b]); whole passes until ~budget_s of
    # thread time (at most 8 passes)
    wb = np.dtype(workloads.word_dtype(vf)).itemsize
    d1_threads = host_cores
    outs = [np.zeros(w.size, workloads.word_dtype(vf)) for _, _, w in fmts]
    jobs1 = []
    for (name, f, w), o in zip(fmts, outs):
        B = int(f["B"])
        step = max(1, -(-B // (4 * host_cores)))
        jobs1 += [(f, b, min(B, b + step), o) for b in range(0, B, step)]
    passes, dt = 0, 0.0
    with cf.ThreadPoolExecutor(max_workers=d1_threads) as ex:
        while passes < 8 and (passes == 0 or dt * d1_threads < budget_s):
            t0 = time.perf_counter()
            list(ex.map(lambda j: oracle.decode_sequential_blocks(*j), jobs1))
            dt += time.perf_counter() - t0
            passes += 1
    for (name, _, w), o in zip(fmts, outs):
        assert np.array_equal(o, w.reshape(-1)), name
    d1 = {"gbs": wb * elems * passes / dt / 1e9, "threads": d1_threads, "passes": passes, "seconds": round(dt, 2)}

    # D2: every host core on the format blocks of each tensor in turn
    jobs = []
    outs2 = [np.zeros(w.size, workloads.word_dtype(vf)) for _, _, w in fmts]
    for (name, f, w), o in zip(fmts, outs2):
        B = int(f["B"])
        step = max(1, -(-B // (4 * host_cores)))
        jobs += [(f, b, min(B, b + step), o) for b in range(0, B, step)]
    passes2, dt2 = 0, 0.0
    with cf.ThreadPoolExecutor(max_workers=host_cores) as ex:
        while passes2 < 8 and (passes2 == 0 or dt2 * host_cores < 2 * budget_s):
            t0 = time.perf_counter()
            list(ex.map(lambda j: oracle.decode_alg1_range(*j), jobs))
            dt2 += time.perf_counter() - t0
            passes2 += 1
    for (name, _, w), o in zip(fmts, outs2):
        assert np.array_equal(o, w.reshape(-1)), name
    d2 = {"gbs": wb * elems * passes2 / dt2 / 1e9, "threads": host_cores, "passes": passes2,
          "seconds": round(dt2, 2)}
    best = d2 if d2["gbs"] >= d1["gbs"] else d1
    sample = (f"{len(fmts)} tensor(s) of the workload ({elems} elements: " + ", ".join(n for n, _, _ in fmts) +
              f"); D1 sequential decode and D2 Alg. 1 emulation, each with {host_cores} threads over the "
              f"format blocks")
    return {"value": best["gbs"], "unit": UNIT, "cores": best["threads"], "kind": "oracle", "sample": sample,
            "d1": d1, "d2": d2, "host_cores": host_cores, "cpu_model": cpu_model()}


def run_reference(args):
    """--impl reference: the CPU oracle (D1, the sequential decoder) timed as the reference arm on this
    workload, with every host core over the format blocks of a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import concurrent.futures as cf

    import oracle
    oracle.build_oracle()
    name, shape = workloads.CONFIGS[args.config][0]
    w = workloads.gaussian_values(shape, workloads.seed_for(args.config, 0, name), args.vf).reshape(-1)
    w = w[: 1 << 24]                                       # bounded sample per step: 16 Mi elements
    lut_bits = args.lut_bits if args.lut_bits == "mono" else int(args.lut_bits)
    fmt = oracle.encode(w, vf=args.vf, lut_bits=lut_bits)
    cores = os.cpu_count() or 1
    out = np.zeros_like(w)
    B = int(fmt["B"])
    step_b = max(1, -(-B // (4 * cores)))
    jobs = [(fmt, b, min(B, b + step_b), out) for b in range(0, B, step_b)]
    with cf.ThreadPoolExecutor(max_workers=cores) as ex:
        def one():
            list(ex.map(lambda j: oracle.decode_sequential_blocks(*j), jobs))
        for _ in range(args.warmup):
            one()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one()
        dt = time.perf_counter() - t0
    assert np.array_equal(out, w)
    wb = np.dtype(workloads.word_dtype(args.vf)).itemsize
    value = wb * w.size * args.steps / dt / 1e9
    sample = (f"D1 sequential decode of the first {w.size} elements of {args.config}/{name} per step, "
              f"{cores} threads over its format blocks")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "config": {"workload": args.config, "elements_per_step": int(w.size),
                                             "value_format": args.vf},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def selftest_dist(args):
    """--selftest-dist: the bench's multi-rank host logic on CPU (gloo): rank r pretends to produce
    (r + 1) GB of BF16 per step in (10 + r) ms per step; rank 0 prints the aggregate and the shard each
    rank would decode for the 70B (strong) and 405B (weak, shard r of 8) sweeps."""
    from paper_2504_11651_b200 import shard
    rank, world, _ = shard.rank_info()
    shard.init_host_group()
    shard.barrier()
    value, tot, ms = shard.aggregate_rate((rank + 1) * 1e9, (10.0 + rank) * args.steps, args.steps)
    cfg70 = dict(workloads.MODELS["llama70b_model"], block_elems=workloads.config_numel("llama70b_block"))
    cfg405 = dict(workloads.MODELS["llama405b_model"], block_elems=workloads.config_numel("llama405b_block"))
    r70, s70 = shard.model_shard(cfg70, rank, world)
    r405, s405 = shard.model_shard(cfg405, rank, world, weak_shards=8)
    units70 = shard.sum_over_ranks([len(r70)])[0]
    mine = {"rank": rank, "llama70b_units": [r70.start, r70.stop], "llama405b_units": [r405.start, r405.stop]}
    import torch.distributed as dist
    allmine = [None] * world
    if world > 1:
        dist.all_gather_object(allmine, mine)
    else:
        allmine = [mine]
    if rank == 0:
        print(json.dumps({"selftest": "dist", "n_ranks": world, "value": value, "unit": UNIT,
                          "bf16_bytes_all_ranks_per_step": tot, "max_ms": ms, "llama70b_units_total": units70,
                          "scaling": {"llama70b_model": s70, "llama405b_model": s405}, "ranks": allmine}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.selftest_dist:
        selftest_dist(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2504_11651_b200 import df11, shard

    rank, world, local = shard.rank_info()
    oversub = os.environ.get("DF11_BENCH_OVERSUBSCRIBE") == "1" and local >= torch.cuda.device_count()
    if oversub:                                  # functional check of the N-rank path on fewer GPUs only
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shard.init_host_group()                      # gloo on the host; NCCL is never initialised
    barrier = shard.barrier
    nvml = shard.nvml_index(dev)

    if args.config in workloads.MODELS:
        run_model(args, df11, dev, rank, world, nvml, barrier)
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- this rank's shard: one transformer block (seeded by rank -> distinct weights per GPU)
    tensors = workloads.config_tensors(args.config, layer=rank, dist=args.dist, vf=args.vf)
    lut_bits = args.lut_bits if args.lut_bits == "mono" else int(args.lut_bits)
    wnp = _word_np(args.vf)
    wtorch = torch.int16 if wnp is np.int16 else torch.uint8
    # host encoder threads: share the host's cores among the ranks of this node
    enc_threads = max(1, (os.cpu_count() or 1) // int(os.environ.get("LOCAL_WORLD_SIZE", str(world))))
    fT, fn = (int(v) for v in args.format.split("x"))
    hs = [df11.encode(w, T=fT, n=fn, num_threads=enc_threads, vf=args.vf, lut_bits=lut_bits) for _, w in tensors]
    N = sum(h.num_elements for h in hs)
    wb = df11.VALUE_FORMATS[args.vf][1]                                    # bytes per decoded word
    upv = 16 // wb                                                         # words per 16 bytes
    scratch = torch.empty(N + 16 * len(hs) + 64, dtype=df11.out_dtype(args.vf), device=dev)   # reused
    outs, o = [], 0
    for h in hs:
        outs.append(scratch[o:o + h.num_elements])
        o += (h.num_elements + upv - 1) // upv * upv                       # keep views 16-byte aligned
    assert o <= scratch.numel()
    dts = [df11.to_device(h, dev) for h in hs]
    plan = df11.BlockPlan(dts, outs)
    kernel_used = args.kernel
    if args.kernel == "auto":
        try:
            plan.run(kernel="fast")
            kernel_used = "fast"
        except df11.Df11Error:
            kernel_used = "alg1"
    # ---- verify once: bit-exact against the original weights (kept on the GPU for the check)
    plan.run(kernel=kernel_used)
    torch.cuda.synchronize()
    for (name, w), out in zip(tensors, plan.outputs()):
        ref = torch.from_numpy(w.reshape(-1).view(wnp)).to(dev)
        if not torch.equal(out.reshape(-1).view(wtorch), ref):
            raise SystemExit(f"bit-exact check failed on {name}")
        del ref
    bf16_bytes = wb * N                                                    # decoded words written
    algo_bytes = sum(dt.compressed_bytes for dt in dts) + bf16_bytes       # read DF11 + write BF16
    # ---- L2: a step that moves less than 4x L2 would be served partly from L2 when repeated, so the
    # timed steps rotate over device copies of the DF11 arrays and outputs (SURVEY 8(d) timing step 2)
    l2 = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20) or (126 << 20))
    copies = 1 if algo_bytes >= 4 * l2 else min(32, -(-4 * l2 // algo_bytes))
    plans = [plan]
    for c in range(1, copies):
        cdts = [df11.clone_device_tensor(d) for d in dts]
        cscratch = torch.empty_like(scratch)
        couts, o = [], 0
        for h in hs:
            couts.append(cscratch[o:o + h.num_elements])
            o += (h.num_elements + upv - 1) // upv * upv
        cp = df11.BlockPlan(cdts, couts)
        cp.run(kernel=kernel_used)
        torch.cuda.synchronize()
        for (name, w), out in zip(tensors, cp.outputs()):
            if not torch.equal(out.reshape(-1).view(wtorch),
                               torch.from_numpy(w.reshape(-1).view(wnp)).to(dev)):
                raise SystemExit(f"bit-exact check failed on copy {c} of {name}")
        plans.append(cp)
    l2_note = (f"inputs larger than L2: {algo_bytes / 1e6:.0f} MB moved per step vs {l2 / 1e6:.0f} MB L2"
               if copies == 1 else
               f"L2 defeated: the timed steps rotate over {copies} device copies of the block "
               f"({copies * algo_bytes / 1e6:.0f} MB >= 4x the {l2 / 1e6:.0f} MB L2; {algo_bytes / 1e6:.0f} MB per step)")

    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        plans[i % copies].run(stream, kernel_used)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    df11.launch_count(reset=True)
    with ClockSampler(nvml) as clocks:
        # the timed region: K back-to-back C-ABI calls bracketed by two events (events between the
        # launches would add ~5 us of gap per launch: scripts/timing_modes.py)
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            plans[(args.warmup + i) % copies].run(stream, kernel_used)
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = df11.launch_count()
    barrier()
    # whole job: sum of every rank's BF16 bytes / the slowest rank's time (gloo reductions on the host)
    value, tot_bf16, total_ms = shard.aggregate_rate(bf16_bytes, t_start.elapsed_time(t_end), args.steps)
    avg_launch_ms = total_ms / args.steps                  # average launch duration over the timed region
    # diagnostic pass (not timed for the headline): per-launch CUDA-event durations
    kd = min(args.steps, 50)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(kd)]
    for i in range(kd):
        ev[i][0].record(stream)
        plans[(args.warmup + i) % copies].run(stream, kernel_used)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    launch_ms = [a.elapsed_time(b) for a, b in ev]

    peak, peak_src = measured_peaks()
    achieved = algo_bytes / (avg_launch_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(args.config, kernel_used + variant_key(args)),
                "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu "
                                  "--set full capture (profiles/ncu_summary.json), not measured in this run",
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": algo_bytes,
                "frac_of_nominal_8tbs": achieved / 8000.0,
                "avg_launch_us": avg_launch_ms * 1e3,
                "launch_us_event_pass": {"launches": kd, "mean": float(np.mean(launch_ms)) * 1e3,
                                         "median": float(np.median(launch_ms)) * 1e3,
                                         "min": float(np.min(launch_ms)) * 1e3,
                                         "p90": float(np.percentile(launch_ms, 90)) * 1e3},
                "note": "achieved = (DF11 bytes read + BF16 bytes written) per launch / the average launch "
                        "duration over the timed region (CUDA events around the K back-to-back launches, slowest "
                        "rank); consecutive launches overlap (programmatic dependent launch: the next "
                        "decode's table build and first tile run under the previous decode's tail, its "
                        "writes wait for it); launch_us_event_pass: a separate pass with events around "
                        "every launch, which serialises them"}

    # ---- the same K steps captured in ONE CUDA graph and replayed (the C ABI is graph-capturable):
    # shorter launch gaps; reported beside the eager headline, not instead of it
    graph = None
    if not args.no_graph:
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for i in range(args.steps):
                plans[(args.warmup + i) % copies].run(gs, kernel_used)
        with torch.cuda.stream(gs):                      # replay() launches on the current stream
            g.replay()
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ga.record(gs)
            g.replay()
            gb.record(gs)
            torch.cuda.synchronize()
        gval, _, gms = shard.aggregate_rate(bf16_bytes, ga.elapsed_time(gb), args.steps)
        graph = {"value": gval, "unit": UNIT, "ms_per_step": gms / args.steps,
                 "what": "the same K block decodes captured in one CUDA graph and replayed (no launch gaps)"}
        del g

    # ---- e2e: through the C ABI with host buffers (pinned H2D of the DF11 arrays, decode, D2H of BF16)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(df11, hs, dts, dev, args.e2e_steps, barrier, tensors, args.vf)

    # ---- NEXT-2: CPU->GPU transfer of the same BF16 bytes (the paper's comparator)
    transfer = None
    if not args.no_transfer:
        transfer = run_transfer(tensors, dev, barrier, value, wnp)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            cpu = oracle_decode_rate(tensors, vf=args.vf, lut_bits=lut_bits)
        except Exception as exc:                                           # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "oracle", "sample": f"failed: {exc}"}

    oversub_any = shard.max_over_ranks([1.0 if oversub else 0.0])[0] > 0
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": args.config, "dist": args.dist, "tensors": len(hs), "elements_per_gpu": N,
                       ("bf16_bytes_per_gpu" if args.vf == "bf16" else "out_bytes_per_gpu"): bf16_bytes,
                       "df11_bytes_per_gpu": algo_bytes - bf16_bytes,
                       "bits_per_weight": 8 * (algo_bytes - bf16_bytes) / N, "T": hs[0].T, "n": hs[0].n,
                       "format": args.format, "value_format": args.vf, "lut_bits": hs[0].lut_bits,
                       "kernel": kernel_used, "parallelism": f"shard{world} (one block per GPU, no collective)",
                       "bf16_bytes_all_ranks_per_step": tot_bf16, "l2": l2_note, "l2_copies": copies},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "graph": graph,
            "transfer_baseline": transfer,
            "gpu_launches": launches,
            **({"oversubscribed": "ranks share GPUs (DF11_BENCH_OVERSUBSCRIBE): a functional check, not a "
                                  "throughput"} if oversub_any else {}),
            "clocks": clocks.summary(),
            "per_gpu_gbs": value / world,
            "env": run_env(dev),
        }
        line["config"].update({"k": [h.k for h in hs], "max_code_len": [h.max_code_len for h in hs],
                               "lut_entry_bytes": [h.lut_entry_bytes for h in hs]})
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_transfer(tensors, dev, barrier, decode_gbs, wnp=np.int16):
    """Pinned host -> device copy of the block's BF16 weights (what DF11 decode replaces when weights
    are offloaded to CPU memory).  Returns GB/s of BF16 delivered and the decode/transfer ratio."""
    import torch
    import torch.distributed as dist
    host = [torch.from_numpy(w.reshape(-1).view(wnp)).pin_memory() for _, w in tensors]
    dst = [torch.empty_like(h, device=dev) for h in host]
    stream = torch.cuda.current_stream()
    for h, d in zip(host, dst):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    a.record(stream)
    for _ in range(reps):
        for h, d in zip(host, dst):
            d.copy_(h, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    from paper_2504_11651_b200 import shard
    nbytes = sum(h.numel() * h.element_size() for h in host)
    gbs, _, _ = shard.aggregate_rate(nbytes * reps, a.elapsed_time(b), 1)
    return {"h2d_gbs": gbs, "unit": UNIT, "decode_over_transfer": decode_gbs / gbs,
            "what": "pinned H2D of the block's BF16 weights vs DF11 decode of the same weights on the GPU"}


def run_model(args, df11, dev, rank, world, nvml, barrier):
    """Whole-model sweeps (BASELINE configs[2] and [4]): the model's transformer blocks (+ embedding,
    LM head) are placed on ranks by plan_shards; a step decodes every block of this rank's shard, one
    df11_decompress_block launch per block into a reused BF16 scratch.

    llama70b_model: the full 80-block model split over the N ranks (strong scaling).
    llama405b_model: the 8-GPU shard set; rank r decodes shard r of 8 whatever N is (weak scaling).
    Weights: `--unique-blocks` distinct blocks per rank are generated (torch Philox on the GPU), host-
    encoded and verified; the rest of the shard are device copies of them (same sizes and entropy)."""
    import torch
    import torch.distributed as dist

    from paper_2504_11651_b200.shard import model_shard, model_units
    m = workloads.MODELS[args.config]
    block_cfg = m["block"]
    shapes = workloads.CONFIGS[block_cfg]
    cfg = dict(m, block_elems=sum(int(np.prod(sh)) for _, sh in shapes))
    units = model_units(cfg)                                               # embed, blocks..., lm_head
    # 405B: the 8-GPU shard set, rank r decodes shard r of 8 (weak); 70B: the model over N ranks (strong)
    rng, scaling = model_shard(cfg, rank, world, weak_shards=8 if args.config == "llama405b_model" else 0)
    mine = list(rng)
    t0 = time.perf_counter()
    # unique encoded units of this rank: up to U blocks + the head/embedding if present
    kinds = []
    for u in mine:
        kinds.append("embed" if u == 0 else ("head" if u == len(units) - 1 else "block"))
    uniq_blocks = min(args.unique_blocks, kinds.count("block"))

    def encode_unit(kind, idx):
        if kind == "block":
            ts = [(name, workloads.gaussian_bf16_torch(sh, workloads.seed_for(block_cfg, idx, name), dev))
                  for name, sh in shapes]
        else:
            ts = [(kind, workloads.gaussian_bf16_torch((m["vocab"], m["hidden"]),
                                                        workloads.seed_for(args.config, idx, kind), dev))]
        threads = max(1, (os.cpu_count() or 1) // int(os.environ.get("LOCAL_WORLD_SIZE", str(world))))
        hs = [df11.encode(w, num_threads=threads) for _, w in ts]
        dts = [df11.to_device(h, dev) for h in hs]
        return ts, hs, dts

    protos = []           # (kind, [DeviceTensor]) verified prototypes
    maxN = 0
    verified = 0
    for i in range(uniq_blocks):
        ts, hs, dts = encode_unit("block", mine[kinds.index("block")] + i)
        protos.append(("block", ts, dts))
    for kind in ("embed", "head"):
        if kind in kinds:
            ts, hs, dts = encode_unit(kind, mine[kinds.index(kind)])
            protos.append((kind, ts, dts))
    for _, ts, dts in protos:
        maxN = max(maxN, sum(dt.num_elements + 8 for dt in dts))
    scratch = torch.empty(maxN + 64, dtype=torch.bfloat16, device=dev)

    def views(dts):
        outs, o = [], 0
        for dt in dts:
            outs.append(scratch[o:o + dt.num_elements])
            o += (dt.num_elements + 7) // 8 * 8
        return outs

    # verify every prototype bit-exactly, then build the per-unit plans (device copies for the rest)
    for kind, ts, dts in protos:
        plan = df11.BlockPlan(dts, views(dts))
        plan.run()
        torch.cuda.synchronize()
        for (name, w), out in zip(ts, plan.outputs()):
            ref = torch.from_numpy(w.reshape(-1).view(np.int16)).to(dev)
            if not torch.equal(out.reshape(-1).view(torch.int16), ref):
                raise SystemExit(f"bit-exact check failed on {kind}/{name}")
            verified += w.size
    block_protos = [dts for kind, _, dts in protos if kind == "block"]
    plans, keep = [], []
    nb = 0
    bf16_bytes = algo = 0
    for kind in kinds:
        if kind == "block":
            src = block_protos[nb % len(block_protos)]
            if nb < len(block_protos):
                dts = src
            else:                                   # device copy of a verified prototype
                dts = [df11.clone_device_tensor(d, out=d.out) for d in src]
                keep.append(dts)
            nb += 1
        else:
            dts = [d for k, _, dd in protos if k == kind for d in dd]
        plans.append(df11.BlockPlan(dts, views(dts)))
        bf16_bytes += sum(2 * d.num_elements for d in dts)
        algo += sum(d.compressed_bytes + 2 * d.num_elements for d in dts)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for p in plans:
            p.run(stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    df11.launch_count(reset=True)
    with ClockSampler(nvml) as clocks:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            for p in plans:
                p.run(stream)
        b.record(stream)
        torch.cuda.synchronize()
    launches = df11.launch_count()
    barrier()
    from paper_2504_11651_b200.shard import aggregate_rate, sum_over_ranks
    value, tot_bf16, ms = aggregate_rate(bf16_bytes, a.elapsed_time(b), args.steps)
    tot_algo = sum_over_ranks([algo])[0]
    peak, peak_src = measured_peaks()
    achieved = algo * args.steps / (a.elapsed_time(b) / 1e3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": args.config, "units_this_rank": len(mine), "blocks_this_rank": kinds.count("block"),
                       "unique_blocks_encoded": uniq_blocks, "bf16_bytes_all_ranks_per_step": tot_bf16,
                       "df11_bytes_all_ranks_per_step": tot_algo - tot_bf16,
                       "parallelism": f"{'shard8' if scaling == 'weak' else 'shard' + str(world)} "
                                      "(contiguous blocks per GPU, no collective)",
                       "setup_s": round(setup_s, 1), "verified_elements_rank0": verified,
                       "l2": "inputs larger than L2 (GB per step)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "peak_source": peak_src,
                         "note": "rank-0 achieved = (DF11 read + BF16 written) / rank-0 step time; one launch per unit"},
            "gpu_launches": launches, "clocks": clocks.summary(), "per_gpu_gbs": value / world,
        }), flush=True)


def run_e2e(df11, hs, dts, dev, steps, barrier, tensors, vf="bf16"):
    import torch

    from paper_2504_11651_b200 import shard
    stream = torch.cuda.current_stream()
    pinned_in, host_views, host_outs = [], [], []
    for h in hs:
        arrs = h.arrays()
        keep = {}
        for key in ("luts", "encoded_exponent", "packed_sign_mantissa", "gaps", "block_output_pos"):
            a = np.ascontiguousarray(arrs[key]).view(np.uint8)
            t = torch.empty(max(a.size, 1), dtype=torch.uint8, pin_memory=True)
            t[: a.size].copy_(torch.from_numpy(a))
            keep[key] = t
        c = df11.HostTensorC()
        import ctypes
        ctypes.memmove(ctypes.byref(c), ctypes.byref(h._c), ctypes.sizeof(c))
        c.luts = ctypes.cast(keep["luts"].data_ptr(), ctypes.POINTER(ctypes.c_uint8))
        c.encoded_exponent = ctypes.cast(keep["encoded_exponent"].data_ptr(), ctypes.POINTER(ctypes.c_uint8))
        c.packed_sign_mantissa = ctypes.cast(keep["packed_sign_mantissa"].data_ptr(), ctypes.POINTER(ctypes.c_uint8))
        c.gaps = ctypes.cast(keep["gaps"].data_ptr(), ctypes.POINTER(ctypes.c_uint8))
        c.block_output_pos = ctypes.cast(keep["block_output_pos"].data_ptr(), ctypes.POINTER(ctypes.c_uint32))
        pinned_in.append(keep)
        host_views.append(c)
        host_outs.append(torch.empty(max(h.num_elements, 1), dtype=df11.out_dtype(vf), pin_memory=True))
    wb = df11.VALUE_FORMATS[vf][1]
    h2d = sum(dt.staging_bytes() for dt in dts)
    d2h = sum(wb * h.num_elements for h in hs)
    N = sum(h.num_elements for h in hs)

    import ctypes
    n = len(hs)
    H = (df11.HostTensorC * n)(*host_views)
    D = (df11.DeviceTensorC * n)(*[dt.descriptor() for dt in dts])
    O = (ctypes.c_void_p * n)(*[ho.data_ptr() for ho in host_outs])
    copy_stream = torch.cuda.Stream()

    def step():
        # one C-ABI call per block: H2D + decode of tensor i+1 overlap the D2H of tensor i
        st = df11.lib().df11_decompress_host_block(H, D, O, n, ctypes.c_void_p(stream.cuda_stream),
                                                   ctypes.c_void_p(copy_stream.cuda_stream))
        if st != 0:
            raise df11.Df11Error(st, df11.lib().df11_last_error_message().decode())

    step()
    torch.cuda.synchronize()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        step()
    b.record(stream)
    torch.cuda.synchronize()
    # the last step's host output must be the original weights
    for ho, h, (name, w) in zip(host_outs, hs, tensors):
        got = ho[: h.num_elements].view(torch.int16 if wb == 2 else torch.uint8).numpy()
        if not np.array_equal(got.view(workloads.word_dtype(vf)), w.reshape(-1)):
            raise SystemExit(f"e2e bit-exact check failed on {name}")
    value, _, _ = shard.aggregate_rate(wb * N, a.elapsed_time(b), steps)
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": steps, "path": "df11_decompress_host_block (pinned H2D + decode on one stream, D2H overlapped on a second)"}


if __name__ == "__main__":
    main()
