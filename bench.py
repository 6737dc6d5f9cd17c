#!/usr/bin/env python3
"""Benchmark of the B200 acquisition hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): 64 tag codes per GPU over 1 s of
synthetic 8 Ms/s I/Q (11 searching windows of 800,000 samples, advance
720,000) x the full frequency-offset sweep (9 lo_freq bins, -400..+400 kHz).
One step = one pass of the hot path over that second of stream:
demodulation of 11 x 9 windows, 6,336 tag-code correlations (argmax,
refinement, statistics, decisions).  Metric: tag-code correlations/s (whole
job), plus the real-time factor.

  value  device-timed, int16 stream already resident in HBM
         (tdg_demodulate_device + tdg_detect, detections left on device)
  e2e    through the C-ABI tdg_search() from PINNED HOST int16 (H2D of the
         stream and D2H of every Detection record inside the timed region)

Multi-GPU (torchrun): weak scaling by tag set -- rank r owns codes
[64r, 64r+64) of the roster and searches the same stream; the per-step
detection lists are gathered over NCCL inside the e2e region.
`--impl reference` times the reference CPU implementation (oracle/_ref, all
host threads) on a bounded sample of the same workload.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_CODES = 64
W = 800000
ADV = 720000
BINS = np.arange(-400e3, 400e3 + 1.0, 100e3)
DURATION = 1.0
FS = 8.0e6
WAVE_PAIRS = 8    # the library's default correlation wave (tdg_set_option "wave_pairs")
N_WIN = int((DURATION * FS - W) // ADV) + 1          # 11
CORR_LEN = 870912
NONZERO = 65741
# algorithmic bytes per correlation with B bins sharing each
# code half-spectrum read, plus the per-(window, bin) input amortised over C.
B_CODE_HALF = 8 * (CORR_LEN // 2 + 1)                 # 3,483,656
B_REPLICA = 4 * NONZERO                               # 262,964
B_WIN = 4 * W + 8 * W + 8 * (CORR_LEN // 2 + 1)       # 13.08 MB per (window, bin)
FLOP_CORR = 47.6e6                                    # SURVEY 8(d) per correlation


def bytes_per_corr(n_bins, n_codes):
    return B_CODE_HALF / n_bins + B_REPLICA + B_WIN / n_codes


def fp32_roof(achieved_tflops, clocks):
    """The stage's real bound: FP32 issue.  Nominal FP32 peak = SMs x 128 lanes
    x 2 flop (FMA) x the median SM clock measured during the timed region."""
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    peak = sms * 128 * 2 * mhz * 1e6 / 1e12
    return {"achieved_tflops": achieved_tflops, "peak_tflops": peak, "frac": achieved_tflops / peak,
            "peak_source": "nominal %d SMs x 128 FP32 lanes x 2 at the measured %.0f MHz median" % (sms, mhz),
            "note": "SURVEY 8(d) 47.6 MFLOP/correlation (5 N log2 N convention) over the correlation stage; "
                    "the stage is FP32-issue / latency bound, not HBM bound (DESIGN.md section 4)"}


def peaks():
    p = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md: 6.65 TB/s)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p = {"hbm_gbs": float(m["hbm_gbs"]), "sm_max_mhz": float(m.get("sm_max_mhz", 1965.0)),
             "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        pass
    return p


class Clocks:
    """nvidia-smi sampling (B200_PROFILING.md clocks line).  The sampler is
    started before the warm-up (nvidia-smi needs ~0.1-0.3 s to produce its
    first sample) and only the samples whose timestamps fall inside the
    timed region (mark_start/mark_end, host clock) are summarised."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]
            self.proc = None

    def summary(self):
        import datetime
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 10 or f[1] != str(self.index):
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            if self.t0 is not None and not (self.t0 - 0.025 <= ts <= self.t1 + 0.025):
                continue
            try:
                sm.append(float(f[2]))
                mx = float(f[3])
            except ValueError:
                continue
            for nm, v in zip(names, f[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "window_s": (self.t1 - self.t0) if self.t0 is not None else None}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# BASELINE.json configs: (codes per GPU, roster size, own stream per rank?)
WORKLOADS = {
    # configs[1]: 64 tag codes per GPU, tag set sharded, one shared stream
    "search": dict(per_gpu=lambda world: N_CODES, roster=lambda world: N_CODES * world, own_stream=False,
                   text="cfg2: %d tag codes/GPU x 1 s of 8 Ms/s int16 I/Q"),
    # configs[2]: 1024 tag codes sharded across the GPUs, detections gathered
    "roster": dict(per_gpu=lambda world: (1024 + world - 1) // world, roster=lambda world: 1024, own_stream=False,
                   text="cfg3: 1024 tag codes sharded (%d per GPU) x 1 s of 8 Ms/s int16 I/Q"),
    # configs[4]: one I/Q stream per GPU (multi-antenna), 256 codes each
    "streams": dict(per_gpu=lambda world: 256, roster=lambda world: 256, own_stream=True,
                    text="cfg5: one 8 Ms/s int16 I/Q stream per GPU x %d tag codes, 1 s"),
}


def make_inputs(rank, world, workload="search"):
    """This rank's code bits, its stream, the injections and the roster index
    of its first code."""
    from paper_2005_10445_b200 import synth
    wl = WORKLOADS[workload]
    per, roster = wl["per_gpu"](world), wl["roster"](world)
    seed = 7 + (rank if wl["own_stream"] else 0)
    bits_all, iq, inj, truth = synth.cfg2_scene(n_codes=roster, n_inject=16, seed=seed)
    if wl["own_stream"]:
        return bits_all, iq, inj, 0
    lo = min(rank * per, roster)
    return bits_all[lo:min(roster, lo + per)], iq, inj, lo


def run_reference(args):
    """Reference arm: oracle/_ref (the reference compiled in place) on the host."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy
    from paper_2005_10445_b200._abi import demod_config
    if not refpy.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtagdsp_ref.so not built"}))
        return
    cfg = demod_config()
    bits, iq, _, _ = make_inputs(0, 1)
    threads = os.cpu_count() or 1
    n_codes = args.ref_codes
    # bounded sample: 1 window x all 9 bins x n_codes codes
    times = []
    for i in range(args.warmup + args.steps):
        t, dets = refpy.search_bench(iq, 0, cfg, BINS, bits[:n_codes], W, ADV, 1, 0.25, threads, code_chunk=1)
        if i >= args.warmup:
            times.append(t)
    per_step = float(np.mean(times))
    units = 1 * len(BINS) * n_codes
    val = units / per_step
    sample = "1 window x %d bins x %d codes (%d correlations) per step, %d host threads" % (
        len(BINS), n_codes, units, threads)
    line = {
        "impl": "reference", "metric": "tag-code correlations/sec", "value": val, "unit": "corr/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (FFT in f64 shim)",
        "data": "synthetic", "config": workload_config(world),
        "real_time_factor": (N_WIN * ADV / FS) / (N_CODES * len(BINS) * N_WIN / val),
        "paper_perf_ratio": (1.0 / val) / (W / FS),
        "paper_throughput_patterns": int(math.floor(val * (W / FS))),
        "paper_tags_searchable_50pct": int(math.floor(0.5 * val * (W / FS))),
        "cpu_baseline": {"value": val, "unit": "corr/s", "cores": threads, "kind": "reference", "sample": sample,
                         "fft": "oracle/fftw_shim (no libfftw3f on the box)"},
        "e2e": {"value": val, "unit": "corr/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def workload_config(world, workload="search"):
    wl = WORKLOADS[workload]
    per = wl["per_gpu"](world)
    return {"workload": (wl["text"] % per) + " (%d windows of %d, advance %d) x %d lo_freq bins (-400..+400 kHz)" % (
                N_WIN, W, ADV, len(BINS)),
            "codes_per_gpu": per, "roster": wl["roster"](world), "windows": N_WIN, "window_len": W,
            "bins": len(BINS), "corr_len": CORR_LEN,
            "correlations_per_step_per_gpu": per * N_WIN * len(BINS),
            "l2": "working set (223 MB code spectra + 345 MB window spectra) exceeds the 126 MB L2; no flush",
            "parallelism": ("one stream per GPU, %d GPU(s)" if wl["own_stream"] else "tag-set sharding, %d GPU(s)") %
                           world}


def cpu_baseline_sample(bits, iq):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy
    from paper_2005_10445_b200._abi import demod_config
    if not refpy.available():
        return None
    threads = os.cpu_count() or 1
    n_codes = 32
    t, _ = refpy.search_bench(iq, 0, demod_config(), BINS, bits[:n_codes], W, ADV, 1, 0.25, threads, code_chunk=1)
    units = len(BINS) * n_codes
    return {"value": units / t, "unit": "corr/s", "cores": threads, "kind": "reference",
            "sample": "1 window x %d bins x %d codes = %d correlations in %.1f s on %d host threads "
                      "(FFT: oracle/fftw_shim, libfftw3f absent)" % (len(BINS), n_codes, units, t, threads)}


def run_tracking(args):
    """BASELINE configs[3]: tracking tasks (proj/src/scheduler.cpp:89-113,
    recording.cpp:360-378) -- 12 ms windows [toa - 2 ms, toa + 10 ms) at
    8 Ms/s, one code each, in latency-bound batches of 1, 8, 64, 512 tasks
    through tdg_track_device (stream resident on the device, i.e. the
    device-side CircularBuffer; Detection records copied back to the host
    inside the timed call).  Reports tasks/s and per-batch latency
    percentiles (host wall clock around each synchronous call)."""
    import ctypes

    import torch
    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import DETECTION_DTYPE, TRACK_TASK_DTYPE, demod_config
    lib = capi.lib()
    cfg = demod_config()
    bits, iq, inj, _ = make_inputs(rank, world)
    TW, PRE = 96000, 16000
    n = iq.size // 2
    ctx = capi.Context(local)
    cs = capi.CodeSet.prepare(ctx, cfg, TW, bits)
    iq_dev = torch.from_numpy(iq).to(f"cuda:{local}")
    rng = np.random.default_rng(5)
    # predicted arrivals: the injected packets (hits) and random times for
    # the other codes (misses), as the scheduler issues them
    pool = [(int(round(t * FS)) - PRE, ci) for ci, t, _, _ in inj]
    while len(pool) < 4096:
        pool.append((int(rng.integers(0, n - TW)), int(rng.integers(0, N_CODES))))
    pool = [(max(0, min(s0, n - TW)), c) for s0, c in pool]
    res = {}
    for B in (1, 8, 64, 512):
        tasks = np.zeros(B, dtype=TRACK_TASK_DTYPE)
        out = np.zeros(B, dtype=DETECTION_DTYPE)
        lat = []
        reps = max(args.steps, 20) if B < 512 else max(args.steps, 10)
        for r in range(args.warmup + reps):
            sel = [pool[(r * B + i) % len(pool)] for i in range(B)]
            tasks["start"] = [x[0] for x in sel]
            tasks["code_index"] = [x[1] for x in sel]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            capi._check(lib.tdg_track_device(ctx.handle, ctypes.byref(cfg), ctypes.c_void_p(iq_dev.data_ptr()), n, 0,
                                             capi._ptr(tasks), B, cs._h, 0.25, capi._ptr(out)))
            dt = time.perf_counter() - t0
            if r >= args.warmup:
                lat.append(dt)
        lat = np.array(lat)
        res[str(B)] = {"tasks_per_s": B / float(np.mean(lat)), "p50_ms": float(np.percentile(lat, 50) * 1e3),
                       "p99_ms": float(np.percentile(lat, 99) * 1e3), "batches": int(lat.size),
                       "accepted_last_batch": int(out["accepted"].sum())}
    line = {"metric": "tracking tasks/sec", "value": res["512"]["tasks_per_s"], "unit": "tasks/s", "n_gpus": 1,
            "higher_is_better": True, "dtype": "f32", "data": "synthetic (cfg2 scene; 16 injected packets tracked, "
            "other tasks are misses at random predicted times)",
            "config": {"workload": "cfg4: tracking windows W=96000 (2 ms pre + 10 ms post at 8 Ms/s), one code per "
                                   "task, batches of 1/8/64/512", "corr_len_b200": cs.info(0)["corr_len"]},
            "batches": res}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="search", choices=["search", "roster", "streams", "tracking"],
                    help="search: BASELINE configs[1] (the headline line); roster: configs[2]; "
                         "tracking: configs[3]; streams: configs[4]")
    ap.add_argument("--ref-codes", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-step", action="store_true",
                    help="run one extra device step between cudaProfilerStart/Stop (ncu --profile-from-start off)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload == "tracking":
        run_tracking(args)
        return

    import ctypes

    import torch
    rank, local, world = dist_env()
    # TDG_BENCH_BACKEND=gloo: exercise the multi-rank path with several ranks
    # sharing fewer GPUs (collectives on host tensors) -- a test knob only;
    # the driver's multi-GPU runs use NCCL, one rank per GPU
    backend = os.environ.get("TDG_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    coll_dev = f"cuda:{local}" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend)
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import DETECTION_DTYPE, demod_config
    lib = capi.lib()
    cfg = demod_config()
    bits, iq, inj, code0 = make_inputs(rank, world, args.workload)
    n_codes = len(bits)
    n_complex = iq.size // 2
    ctx = capi.Context(local)
    # TDG_BENCH_OPTIONS="wave_pairs=10,n_streams=4": tuning knobs for sweeps
    # (tdg_set_option); the default run sets none
    for kv in filter(None, os.environ.get("TDG_BENCH_OPTIONS", "").split(",")):
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    cs = capi.CodeSet.prepare(ctx, cfg, W, bits)
    corr_len_used = cs.info(0)["corr_len"]
    win = capi.Windows(ctx, W, N_WIN, len(BINS))
    iq_dev = torch.from_numpy(iq).to(f"cuda:{local}")
    iq_pin = torch.from_numpy(iq).pin_memory()
    n_units = n_codes * N_WIN * len(BINS)
    out_pin = torch.empty(n_units * DETECTION_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
    stream = torch.cuda.ExternalStream(ctx.stream(), device=f"cuda:{local}")
    bins = np.ascontiguousarray(BINS)

    def step_device():
        capi._check(lib.tdg_demodulate_device(ctx.handle, win._h, ctypes.byref(cfg), capi._ptr(bins), bins.size,
                                              ctypes.c_void_p(iq_dev.data_ptr()), n_complex, 0, ADV, N_WIN))
        capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, FS, None))

    nout = ctypes.c_uint64()

    # end-to-end = the streaming public API: each step uploads one second of
    # pinned host I/Q into the device-resident CircularBuffer (tdg_ring_push,
    # its own copy stream) and searches that second's windows straight from
    # the ring (tdg_search_ring), Detection records copied back to pinned host
    # memory; the upload of second k+1 overlaps the search of second k.
    ring = capi.Ring(ctx, 3 * n_complex)
    stream_pos = [0]

    def step_e2e():
        start = stream_pos[0]
        capi._check(lib.tdg_ring_push(ring._h, ctypes.c_void_p(iq_pin.data_ptr()), n_complex, start, None))
        capi._check(lib.tdg_search_ring(ctx.handle, ring._h, ctypes.byref(cfg), capi._ptr(bins), bins.size, start, W,
                                        ADV, N_WIN, cs._h, 0.25, ctypes.c_void_p(out_pin.data_ptr()), n_units,
                                        int(world > 1)))
        stream_pos[0] += n_complex
        if world > 1:
            # the path's one exchange: every rank's accepted detections, all-gathered over NCCL
            from paper_2005_10445_b200 import dist as tdist
            recs = np.frombuffer(out_pin.numpy().tobytes(), dtype=DETECTION_DTYPE)
            tdist.gather_detections(recs, code0, device=coll_dev, accepted_only=True)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        ctx.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region ---------------------------------------
    clk = Clocks(local).start()
    for _ in range(args.warmup):
        step_device()
    barrier()
    launches0 = capi.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    clk.mark_start()
    ev0.record(stream)
    for _ in range(args.steps):
        step_device()
    ev1.record(stream)
    barrier()
    clk.mark_end()
    clk.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = (capi.kernel_launches() - launches0) // args.steps
    ms_max = max_over_ranks(ms)
    value = n_units * world / (ms_max / 1e3)

    if args.profile_step:
        torch.cuda.cudart().cudaProfilerStart()
        step_device()
        barrier()
        torch.cuda.cudart().cudaProfilerStop()

    # ---- end-to-end through the C-ABI from pinned host memory ----------------
    for _ in range(args.warmup):
        step_e2e()
    barrier()
    t0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(args.steps):
        step_e2e()
    ev1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    wall_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / args.steps)
    e2e = n_units * world / (e2e_ms / 1e3)

    # ---- per-kernel CUDA events (same steps, separate pass: recording an
    # event pair around each of ~800 launches perturbs the step time) -------
    ctx.kernel_time_reset()
    ctx.set_option("time_kernels", 1)
    for _ in range(args.steps):
        step_device()
    barrier()
    kt = {k: ctx.kernel_time(k) for k in ("demod", "fwd_pass1", "fwd_pass2", "corr", "stats")}
    ctx.set_option("time_kernels", 0)

    # ---- roofline of the dominant stage: the correlation engine -------------
    # (k_corr_pass pass A + pass B on overlapped streams, one per-step event pair)
    pk = peaks()
    n_corr_launch, ms_corr = kt["corr"]
    corr_ms_step = ms_corr / max(1, n_corr_launch)
    bpc = bytes_per_corr(len(BINS), n_codes)
    achieved = bpc * n_units / (corr_ms_step / 1e3) / 1e9
    total_ms = sum(v[1] for v in kt.values())
    shares = {k: round(v[1] / total_ms, 4) if total_ms else None for k, v in kt.items()}
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = tj["corr_dram_bytes_per_step"]
    except Exception:
        pass

    if rank != 0:
        return
    cpu = None if args.no_cpu_baseline else cpu_baseline_sample(bits, iq)
    clocks = clk.summary()
    line = {
        "metric": "tag-code correlations/sec", "value": value, "unit": "corr/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy scene: 16 of the codes injected at known fractional delays, offsets "
                "U(-200,200) kHz, SNR {0,5,10,20} dB in 10 dB noise; int16 at scale 8192)",
        "config": dict(workload_config(world, args.workload), corr_len_b200=corr_len_used),
        # stream seconds searched per wall second for the whole roster (64 x
        # n_gpus codes) x 9 bins: N_WIN windows x advance per step
        "real_time_factor": (N_WIN * ADV / FS) / (ms_max / 1e3),
        "real_time_factor_e2e": (N_WIN * ADV / FS) / (e2e_ms / 1e3),
        # the paper's figures (proj/src/harness.cpp:15-25): perf_ratio = time
        # per pattern (one code against one window, here per bin) / window
        # duration, and the patterns one GPU keeps up with in real time
        # (search_share 1) = floor(1 / perf_ratio); from the e2e time
        "paper_perf_ratio": (e2e_ms / 1e3 / n_units) / (W / FS),
        "paper_throughput_patterns": int(math.floor(1.0 / ((e2e_ms / 1e3 / n_units) / (W / FS)))),
        # PAPER Table 3's column (search_share 0.5): 6 / 26 / 77 / 315 tags on
        # i7-8700T / Jetson TX2 / GTX 1050 / Titan Xp
        "paper_tags_searchable_50pct": int(math.floor(0.5 / ((e2e_ms / 1e3 / n_units) / (W / FS)))),
        "e2e": {"value": e2e, "unit": "corr/s", "ms_per_step": e2e_ms, "wall_ms_per_step": wall_ms,
                "h2d_bytes_per_step": int(iq.nbytes), "d2h_bytes_per_step": int(n_units * DETECTION_DTYPE.itemsize),
                "path": "streaming C-ABI: tdg_ring_push (pinned host int16 -> device CircularBuffer, copy "
                        "stream) + tdg_search_ring (Detection records -> pinned host), upload of step k+1 "
                        "overlapping the search of step k"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm",
                     "kernel": "correlation engine per step: k_corr_pass<27,32,32,32,0> (spectral product + "
                               "first inverse-FFT pass) and k_corr_pass<...,1> (second pass + argmax), "
                               "%d launches in waves of %d pairs over 6 pass-A + 6 pass-B streams" % (
                                   2 * (((n_codes + 1) // 2 * N_WIN * len(BINS) + WAVE_PAIRS - 1) // WAVE_PAIRS),
                                   WAVE_PAIRS),
                     "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                     "traffic": traffic, "peak_source": pk["source"],
                     "traffic_note": "dram__bytes_read+write of all correlation launches of one step, warm L2 "
                                     "(ncu --cache-control none, profiles/traffic.json)",
                     "algorithmic_bytes_per_corr": bpc, "corr_per_step": n_units, "stage_ms_per_step": corr_ms_step,
                     "fp32": fp32_roof(n_units * FLOP_CORR / (corr_ms_step / 1e3) / 1e12, clocks)},
        "kernel_ms_per_step": {k: v[1] / args.steps for k, v in kt.items()},
        "kernel_share": shares,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
