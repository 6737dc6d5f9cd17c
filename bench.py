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
  e2e    the streaming C-ABI from PINNED HOST int16: tdg_ring_push of the
         step's second into the device CircularBuffer + tdg_search_ring with
         every Detection record copied back to pinned host memory (H2D and
         D2H inside the timed region)

Nothing is timed before a correctness gate passes (the reference's run_bench
gate, proj/src/harness.cpp:58-73): the injected packets found at the right
ToA, no absent code accepted, and window 0 x 9 bins x 32 codes equal to the
reference's records (oracle/_ref) under the parity contract.

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


def roofline(n_units, stage_ms, fp32_peak_tflops, hbm_peak_gbs, bytes_corr, flop_corr=FLOP_CORR):
    """SURVEY 8(d) roofline of the correlation stage: bound = FP32 (the
    stage's arithmetic intensity sits at the FP32 ridge and the bin sweep
    shares every code read), achieved = flops per correlation x correlations /
    stage time, frac = achieved / peak; attainable corr/s = min(HBM peak /
    bytes per corr, FP32 peak / flops per corr); the HBM fraction is kept as
    a secondary figure."""
    t = stage_ms / 1e3
    achieved = n_units * flop_corr / t / 1e12
    attainable = min(hbm_peak_gbs * 1e9 / bytes_corr, fp32_peak_tflops * 1e12 / flop_corr)
    hbm = bytes_corr * n_units / t / 1e9
    return {"bound": "fp32", "achieved": achieved, "peak": fp32_peak_tflops, "unit": "TFLOP/s",
            "frac": achieved / fp32_peak_tflops, "attainable_corr_per_s": attainable,
            "stage_corr_per_s": n_units / t, "frac_of_attainable": (n_units / t) / attainable,
            "hbm": {"achieved": hbm, "peak": hbm_peak_gbs, "unit": "GB/s", "frac": hbm / hbm_peak_gbs,
                    "algorithmic_bytes_per_corr": bytes_corr}}


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


def cpu_model():
    """CPU model, logical CPU count and max MHz from lscpu (the box's host)."""
    info = {"model": None, "logical_cpus": os.cpu_count(), "max_mhz": None}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for l in out.splitlines():
            k, _, v = l.partition(":")
            v = v.strip()
            if k.strip() == "Model name":
                info["model"] = v
            elif k.strip() in ("CPU max MHz", "CPU MHz") and info["max_mhz"] is None:
                info["max_mhz"] = float(v)
    except Exception:
        pass
    return info


def reference_sample(bits, iq, n_codes, n_bins, threads, code_chunk=2):
    """The reference's own searching loop (proj/src/recording.cpp:277-286: one
    demodulate_window per (window, bin) shared by every code, then detect over
    the codes) on window 0 of the stream, `n_bins` lo_freq bins x `n_codes`
    codes, on `threads` host threads (oracle/_ref, tdref_search_bench_shared).
    Returns (seconds, records [bin][code], stage thread-seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy
    from paper_2005_10445_b200._abi import demod_config
    t, recs, st = refpy.search_bench_shared(iq[:2 * W], 0, demod_config(), BINS[:n_bins], bits[:n_codes], W, ADV, 1,
                                            0.25, threads, code_chunk=code_chunk)
    return t, recs.reshape(n_bins, n_codes), st


def single_core_sample(bits, iq):
    """One host core: 1 window x 1 bin x 8 codes through the same loop."""
    t, _, st = reference_sample(bits, iq, 8, 1, 1, code_chunk=8)
    return {"value": 8 / t, "unit": "corr/s", "cores": 1, "sample": "1 window x 1 bin x 8 codes (%.2f s)" % t,
            "stage_s": st}


def stage_split(st):
    tot = sum(st.values()) or 1.0
    return {k: round(v / tot, 4) for k, v in st.items()}


def run_reference(args):
    """Reference arm: oracle/_ref (the reference compiled in place) on the
    host, like for like with the reference's own loop: one demodulation per
    (window, bin) shared by all codes, detect() over the codes, work spread
    over every host thread."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy
    if not refpy.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtagdsp_ref.so not built"}))
        return
    bits, iq, _, _ = make_inputs(0, 1)
    threads = os.cpu_count() or 1
    n_codes = args.ref_codes
    times, stages = [], {"demod": 0.0, "correlation": 0.0, "peak_stats": 0.0}
    for i in range(args.warmup + args.steps):
        t, _, st = reference_sample(bits, iq, n_codes, len(BINS), threads)
        if i >= args.warmup:
            times.append(t)
            for k in stages:
                stages[k] += st[k]
    per_step = float(np.mean(times))
    units = 1 * len(BINS) * n_codes
    val = units / per_step
    single = single_core_sample(bits, iq)
    cpu = cpu_model()
    sample = ("1 window x %d bins x %d codes (%d correlations) per step: one demodulate_window per (window, bin) "
              "shared by all codes, detect() over chunks of 2 codes, %d host threads" % (len(BINS), n_codes, units,
                                                                                      threads))
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
                         "fft": "oracle/fftw_shim (no libfftw3f on the box)", "cpu": cpu,
                         "single_core": single, "stage_split": stage_split(stages)},
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


def correctness_gate(recs, inj, code0, n_codes, ref_recs, bits, iq):
    """Refuse to time a wrong pipeline (the reference's run_bench gate,
    proj/src/harness.cpp:58-73): every injected packet of this rank's codes
    that lies wholly inside a window is accepted at its nearest lo_freq bin
    with |ToA error| < 0.5 sample, no absent code is accepted anywhere, and
    the records of window 0 x all bins x the CPU sample's codes match the
    reference's (oracle/_ref) under the parity contract (near-ties
    documented with their margin on the reference's own xc).
    recs: this rank's GPU records [window][bin][code]."""
    problems, found, weak = [], 0, [0, 0]
    mine = [(ci - code0, t, g, foff) for ci, t, g, foff in inj if code0 <= ci < code0 + n_codes]
    for c, t, g, foff in mine:
        a = t * FS
        b = int(np.argmin(np.abs(BINS - foff)))
        snr = 10.0 + 20.0 * math.log10(g)   # packet amplitude g over the 10 dB noise floor
        for wi in range(N_WIN):
            s0 = wi * ADV
            if s0 <= a and a + 65536 + 256 <= s0 + W:
                r = recs[wi, b, c]
                hit = bool(r["accepted"]) and abs(float(r["toa_seconds"]) * FS - a) < 0.5
                if snr < 5.0:            # 0 dB packets: reported, not required
                    weak[0] += 1
                    weak[1] += int(hit)
                elif not hit:
                    problems.append(("injection", c + code0, wi, float(r["score"]), float(r["toa_seconds"]) * FS, a))
                else:
                    found += 1
    injected = {c for c, _, _, _ in mine}
    spurious = [(int(w), int(b), int(c)) for w, b, c in zip(*np.nonzero(recs["accepted"])) if int(c) not in injected]
    problems += [("spurious",) + x for x in spurious]
    report = None
    if ref_recs is not None:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import refpy
        from paritycheck import ParityReport, RefSlots
        from paper_2005_10445_b200._abi import demod_config
        nb, nc = ref_recs.shape
        rs = RefSlots(refpy, demod_config(), bits, iq, W)
        report = ParityReport("bench gate: window 0 x %d bins x %d codes" % (nb, nc))
        for b in range(nb):
            bad = rs.compare(recs[0, b, :nc], ref_recs[b], 0, BINS[b], FS, report=report)
            problems += [("parity", b) + tuple(x) for x in bad]
    gate = {"injections_found": found, "injections_expected": found + sum(p[0] == "injection" for p in problems),
            "injections_0db_found": weak[1], "injections_0db": weak[0], "spurious": len(spurious),
            "ok": not problems,
            "rule": "every injected packet >= 5 dB SNR wholly inside a window accepted at its nearest bin with |ToA "
                    "error| < 0.5 sample; no absent code accepted; window 0 x 9 bins x 32 codes equal to oracle/_ref"}
    if report is not None:
        s = report.summary()
        gate["parity"] = {k: s[k] for k in ("records", "peak_index_exact", "near_ties", "mismatches",
                                             "max_delta_accepted_records")}
    return gate, problems


def tracking_probe(ctx, cfg, bits, iq, iq_dev, inj, steps, warmup, with_cpu=True, batches=(1, 8, 64, 512)):
    """BASELINE configs[3]: tracking tasks (proj/src/scheduler.cpp:89-113,
    recording.cpp:360-378) -- 12 ms windows [toa - 2 ms, toa + 10 ms) at
    8 Ms/s, one code each, in latency-bound batches through tdg_track_device
    (stream resident on the device, i.e. the device-side CircularBuffer;
    Detection records copied back to the host inside the timed call).
    Returns per-batch tasks/s and latency percentiles (host wall clock around
    each synchronous call), the reference's CPU figure beside them and the
    parity of 32 tasks against the reference."""
    import ctypes

    import torch
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import DETECTION_DTYPE, TRACK_TASK_DTYPE
    lib = capi.lib()
    TW, PRE = 96000, 16000
    n = iq.size // 2
    cs = capi.CodeSet.prepare(ctx, cfg, TW, bits)
    rng = np.random.default_rng(5)
    # predicted arrivals: the injected packets (hits) and random times for
    # the other codes (misses), as the scheduler issues them
    pool = [(int(round(t * FS)) - PRE, ci) for ci, t, _, _ in inj]
    while len(pool) < 4096:
        pool.append((int(rng.integers(0, n - TW)), int(rng.integers(0, len(bits)))))
    pool = [(max(0, min(s0, n - TW)), c) for s0, c in pool]
    res = {}
    for B in batches:
        tasks = np.zeros(B, dtype=TRACK_TASK_DTYPE)
        out = np.zeros(B, dtype=DETECTION_DTYPE)
        lat = []
        reps = max(steps, 20) if B < 512 else max(steps, 10)
        for r in range(warmup + reps):
            sel = [pool[(r * B + i) % len(pool)] for i in range(B)]
            tasks["start"] = [x[0] for x in sel]
            tasks["code_index"] = [x[1] for x in sel]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            capi._check(lib.tdg_track_device(ctx.handle, ctypes.byref(cfg), ctypes.c_void_p(iq_dev.data_ptr()), n, 0,
                                             capi._ptr(tasks), B, cs._h, 0.25, capi._ptr(out)))
            dt = time.perf_counter() - t0
            if r >= warmup:
                lat.append(dt)
        lat = np.array(lat)
        res[str(B)] = {"tasks_per_s": B / float(np.mean(lat)), "p50_ms": float(np.percentile(lat, 50) * 1e3),
                       "p99_ms": float(np.percentile(lat, 99) * 1e3), "batches": int(lat.size),
                       "accepted_last_batch": int(out["accepted"].sum())}
    # CPU beside it: the reference's tracking task body (demodulate_window +
    # detect against one code prepared for the tracking shape,
    # recording.cpp:360-378) on one host core -- the reference's scheduler is
    # sequential -- over 32 tasks of the same pool, and the GPU's records of
    # those tasks against the reference's (parity contract).
    cpu, parity = None, None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy
    if refpy.available() and with_cpu:
        sel = pool[:32]
        st = np.array([x[0] for x in sel], np.int64)
        co = np.array([x[1] for x in sel], np.uint64)
        t_cpu, want = refpy.track_bench(iq, 0, cfg, bits, TW, st, co, 0.25)
        cpu = {"value": len(sel) / t_cpu, "unit": "tasks/s", "cores": 1, "kind": "reference",
               "sample": "32 tracking tasks (16 injected packets + 16 misses), one at a time on one host core",
               "cpu": cpu_model()}
        got = np.zeros(len(sel), dtype=DETECTION_DTYPE)
        tasks = np.zeros(len(sel), dtype=TRACK_TASK_DTYPE)
        tasks["start"], tasks["code_index"] = st, co
        capi._check(lib.tdg_track_device(ctx.handle, ctypes.byref(cfg), ctypes.c_void_p(iq_dev.data_ptr()), n, 0,
                                         capi._ptr(tasks), len(sel), cs._h, 0.25, capi._ptr(got)))
        from paritycheck import ParityReport, RefSlots
        rep = ParityReport("tracking: 32 tasks")
        bad = []
        rs = RefSlots(refpy, cfg, bits, iq, TW)
        for i in range(len(sel)):
            bad += rs.compare(got[i:i + 1], want[i:i + 1], int(st[i]), cfg.lo_freq, FS, report=rep)
        parity = {"records": rep.records, "peak_index_exact": rep.peak_exact, "near_ties": len(rep.near_ties),
                  "mismatches": len(bad), "accepted": int(got["accepted"].sum())}
        if bad:
            sys.stderr.write(json.dumps({"error": "tracking parity failed", "bad": [str(b) for b in bad[:10]]}) + "\n")
            sys.exit(3)
    corr_len = cs.info(0)["corr_len"]
    cs.close()
    return res, cpu, parity, corr_len


def run_tracking(args):
    """BASELINE configs[3] as its own line (see tracking_probe)."""
    import torch
    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    bits, iq, inj, _ = make_inputs(rank, world)
    ctx = capi.Context(local)
    iq_dev = torch.from_numpy(iq).to(f"cuda:{local}")
    res, cpu, parity, corr_len = tracking_probe(ctx, cfg, bits, iq, iq_dev, inj, args.steps, args.warmup,
                                                with_cpu=not args.no_cpu_baseline)
    line = {"metric": "tracking tasks/sec", "value": res["512"]["tasks_per_s"], "unit": "tasks/s", "n_gpus": 1,
            "higher_is_better": True, "dtype": "f32", "data": "synthetic (cfg2 scene; 16 injected packets tracked, "
            "other tasks are misses at random predicted times)",
            "config": {"workload": "cfg4: tracking windows W=96000 (2 ms pre + 10 ms post at 8 Ms/s), one code per "
                                   "task, batches of 1/8/64/512", "corr_len_b200": corr_len},
            "batches": res, "cpu_baseline": cpu, "parity": parity}
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
    ap.add_argument("--ref-codes", type=int, default=32)
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
        capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, FS, None, 0))

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

    # ---- correctness gate: nothing is timed unless the pipeline is right ----
    gate_recs = capi.search(ctx, cfg, bins, iq, cs, W, ADV).reshape(N_WIN, len(BINS), n_codes)
    cpu, ref_recs = None, None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy
    if rank == 0 and not args.no_cpu_baseline and refpy.available():
        threads = os.cpu_count() or 1
        nref = min(32, n_codes)
        t_ref, ref_recs, st = reference_sample(bits, iq, nref, len(BINS), threads)
        cpu = {"value": len(BINS) * nref / t_ref, "unit": "corr/s", "cores": threads, "kind": "reference",
               "sample": "1 window x %d bins x %d codes = %d correlations in %.2f s on %d host threads: one "
                         "demodulate_window per (window, bin) shared by all codes, detect() over chunks of 2 codes "
                         "(FFT: oracle/fftw_shim, libfftw3f absent)" % (len(BINS), nref, len(BINS) * nref, t_ref,
                                                                         threads),
               "cpu": cpu_model(), "stage_split": stage_split(st)}
    gate, problems = correctness_gate(gate_recs, inj, code0, n_codes, ref_recs, bits, iq)
    if problems:
        sys.stderr.write(json.dumps({"error": "correctness gate failed; not timing", "gate": gate,
                                     "problems": [list(map(str, p)) for p in problems[:20]]}) + "\n")
        sys.exit(3)

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

    # ---- GPU code preparation (prepare_code for the whole
    # set -- synth_replica, demodulation, support/energy, forward transforms of
    # the code pairs), a fresh set of the same codes, outside the timed steps
    prep = []
    for _ in range(3):
        barrier()
        t_prep = time.perf_counter()
        cs2 = capi.CodeSet.prepare(ctx, cfg, W, bits)
        ctx.synchronize()
        prep.append((time.perf_counter() - t_prep) * 1e3)
        cs2.close()
    prep_ms = min(prep)
    code_prep = {"codes": n_codes, "ms": round(prep_ms, 3), "codes_per_s": round(n_codes / (prep_ms / 1e3), 1),
                 "ms_each": [round(x, 2) for x in prep],
                 "note": "wall clock of tdg_codeset_prepare (synchronous; fresh device buffers each time), "
                         "window_len %d, best of 3" % W}

    # ---- tracking (BASELINE configs[3]) on the same box, so its latency and
    # the reference's CPU figure beside it appear in the driver-visible line
    # (outside every timed region of this line; single-rank runs only)
    tracking = None
    if world == 1 and args.workload == "search":
        tres, tcpu, tpar, _ = tracking_probe(ctx, cfg, bits, iq, iq_dev, inj, args.steps, args.warmup,
                                             with_cpu=not args.no_cpu_baseline)
        tracking = {"workload": "cfg4: W=96000 windows, one code per task, tdg_track_device",
                    "p50_ms": {k: round(v["p50_ms"], 4) for k, v in tres.items()},
                    "p99_ms": {k: round(v["p99_ms"], 4) for k, v in tres.items()},
                    "tasks_per_s": {k: round(v["tasks_per_s"], 1) for k, v in tres.items()},
                    "cpu_baseline": tcpu, "parity": tpar}

    # ---- roofline of the dominant stage: the correlation engine -------------
    # (k_corr_pass pass A + pass B on overlapped streams, one per-step event
    # pair).  SURVEY 8(d): the stage is FP32 bound (AI ~12.7 flop/B at the
    # ridge, and the 9-bin sweep shares each code read 9 ways), so the bound
    # is FP32: achieved = 47.6 MFLOP per correlation x correlations per step /
    # stage time; peak = the packed-FFMA2 rate MEASURED on this GPU now
    # (tdg_fp32_peak, the instruction the codelets use); attainable corr/s =
    # min(HBM peak / bytes per corr, FP32 peak / flops per corr).
    pk = peaks()
    n_corr_launch, ms_corr = kt["corr"]
    corr_ms_step = ms_corr / max(1, n_corr_launch)
    bpc = bytes_per_corr(len(BINS), n_codes)
    hbm_achieved = bpc * n_units / (corr_ms_step / 1e3) / 1e9
    ffma_peak, ffma2_peak = capi.fp32_peak(local)
    fp32_peak = max(ffma_peak, ffma2_peak)
    roof = roofline(n_units, corr_ms_step, fp32_peak, pk["hbm_gbs"], bpc)
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
    clocks = clk.summary()
    line = {
        "metric": "tag-code correlations/sec", "value": value, "unit": "corr/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy scene: 16 of the codes injected at known fractional delays, offsets "
                "U(-200,200) kHz, SNR {0,5,10,20} dB in 10 dB noise; int16 at scale 8192)",
        "config": dict(workload_config(world, args.workload), corr_len_b200=corr_len_used),
        "gate": gate,
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
        "code_prep": code_prep,
        "tracking": tracking,
        "roofline": dict(roof, **{
            "kernel": "correlation engine per step: k_corr_pass<27,32,32,32,0> (spectral product + first "
                      "inverse-FFT pass) and k_corr_pass<...,1> (second pass + argmax) in waves over 6 pass-A + 6 "
                      "pass-B streams",
            "traffic": traffic,
            "peak_source": "measured live on this GPU (tdg_fp32_peak): packed FFMA2 %.1f TFLOP/s, scalar FFMA "
                           "%.1f TFLOP/s; peak = the larger" % (ffma2_peak, ffma_peak),
            "flops_per_corr": FLOP_CORR, "corr_per_step": n_units, "stage_ms_per_step": corr_ms_step,
            "traffic_note": "dram__bytes_read+write of all correlation launches of one step (profiles/traffic.json, "
                            "ncu); algorithmic %.4g B/step" % (bpc * n_units),
            "hbm_peak_source": pk["source"]}),
        "kernel_ms_per_step": {k: v[1] / args.steps for k, v in kt.items()},
        "kernel_share": shares,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
