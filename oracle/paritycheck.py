"""TEST INFRASTRUCTURE ONLY (oracle side).  Parity checker: compares B200
Detection records with the reference's (oracle/_ref) under the tolerances the
north star states (BASELINE.json): peak index and accept/partial exact, except
near-ties documented with their margin; ToA, score and correlation magnitudes
within ~1e-4 relative.  Used by tests/ (re-exported by tests/parity.py) and by
bench.py's correctness gate (its cpu_baseline leg), never by the product.

Every comparison can feed a ParityReport, which records the number of records
compared, each near-tie with its margin on the reference's own xc, and the
worst |delta| per field -- the numbers profiles/parity_cfg2.md publishes."""
import json

import numpy as np

REL = 1e-4
NEAR_TIE = 1e-5   # documented near-tie: margin on the reference's xc below this


def direct_xcorr(d, dc):
    """Brute-force lag-domain oracle (test_detector.cpp:38-47), float64."""
    d = np.asarray(d, np.float64)
    dc = np.asarray(dc, np.float64)
    W, n = d.size, dc.size
    full = np.correlate(np.concatenate([d, np.zeros(n)]), dc, mode="valid")[:W]
    return full


def near_tie_margin(xc_ref, j_ref, j_gpu):
    """(|xc[j_ref]| - |xc[j_gpu]|) / |xc[j_ref]| on the reference's own xc."""
    a = abs(float(xc_ref[j_ref]))
    b = abs(float(xc_ref[j_gpu]))
    return (a - b) / a if a else 0.0


def delta_tolerance(xc_ref, j, delta, eps, xc_scale=0.0):
    """Bound on |subsample_offset| differences caused by perturbations of the
    xc values: delta = 0.5(a-c)/(a-2b+c) (detector.cpp:136-145) has
    |d delta| <= e*(1+2|delta|)/|a-2b+c| for an absolute perturbation e of
    a, b, c, plus a 1e-4 floor.  e = eps * max(b, xc_scale): a rounding-level
    difference of the replica or window (two FFT implementations) perturbs
    each lag by ~eps relative to the Cauchy-Schwarz scale sqrt(q*E) =
    |w_c/score| of the dot product, which for a weak (absent-code) peak is
    far above b itself."""
    if xc_ref is None or j == 0 or j + 1 >= len(xc_ref):
        return 1e-4
    a, b, c = (abs(float(xc_ref[j - 1])), abs(float(xc_ref[j])), abs(float(xc_ref[j + 1])))
    den = abs(a - 2.0 * b + c)
    if den == 0.0:
        return 1e-4
    return 1e-4 + eps * max(b, xc_scale) * (1.0 + 2.0 * abs(delta)) / den


def pc_scale(dc, u, j):
    """Cauchy-Schwarz scale of p_c = sum_i dc[i] u[j+i] (detector.cpp:147-165):
    a rounding-level relative perturbation eps of dc and u (two FFT
    implementations in the demodulation) moves p_c by at most about
    eps * sqrt(sum dc^2 * sum u[j:j+n]^2), which for an absent code's residual
    p_c is far above |p_c| itself."""
    dc = np.asarray(dc, np.float64)
    seg = np.asarray(u, np.float64)[j:j + dc.size]
    return float(np.sqrt(np.dot(dc[:seg.size], dc[:seg.size]) * np.dot(seg, seg)))


class ParityReport:
    """Accumulates what a parity run saw: records compared, exact peak
    matches, near-ties (with margins), accepted counts and the worst absolute
    and relative |delta| per field."""

    FIELDS = ("subsample_offset", "toa_samples", "peak_value", "w_c", "q", "p_c", "score")

    def __init__(self, name=""):
        self.name = name
        self.records = 0
        self.peak_exact = 0
        self.accepted_ref = 0
        self.accepted_gpu = 0
        self.near_ties = []       # dicts: key, j_ref, j_gpu, margin, score_ref, accepted
        self.max_abs = {f: 0.0 for f in self.FIELDS}
        self.max_rel = {f: 0.0 for f in self.FIELDS}
        self.max_rel_accepted = {f: 0.0 for f in self.FIELDS}
        self.mismatches = 0

    def field(self, f, g, w, accepted):
        d = abs(float(g) - float(w))
        self.max_abs[f] = max(self.max_abs[f], d)
        if f not in ("subsample_offset", "toa_samples"):
            r = d / abs(float(w)) if float(w) else (0.0 if d == 0 else float("inf"))
            self.max_rel[f] = max(self.max_rel[f], r)
            if accepted:
                self.max_rel_accepted[f] = max(self.max_rel_accepted[f], r)
        elif accepted:
            self.max_rel_accepted[f] = max(self.max_rel_accepted[f], d)

    def merge(self, other):
        self.records += other.records
        self.peak_exact += other.peak_exact
        self.accepted_ref += other.accepted_ref
        self.accepted_gpu += other.accepted_gpu
        self.near_ties += other.near_ties
        self.mismatches += other.mismatches
        for f in self.FIELDS:
            self.max_abs[f] = max(self.max_abs[f], other.max_abs[f])
            self.max_rel[f] = max(self.max_rel[f], other.max_rel[f])
            self.max_rel_accepted[f] = max(self.max_rel_accepted[f], other.max_rel_accepted[f])

    def summary(self):
        return {"name": self.name, "records": self.records, "peak_index_exact": self.peak_exact,
                "near_ties": len(self.near_ties), "mismatches": self.mismatches,
                "accepted_ref": self.accepted_ref, "accepted_gpu": self.accepted_gpu,
                "max_abs_delta": self.max_abs, "max_rel_delta": self.max_rel,
                "max_delta_accepted_records": self.max_rel_accepted,
                "near_tie_list": self.near_ties}

    def markdown(self):
        s = self.summary()
        out = ["### %s" % self.name, "",
               "| records compared | peak index exact | near-ties | mismatches | accepted (ref / B200) |",
               "|---|---|---|---|---|",
               "| %d | %d | %d | %d | %d / %d |" % (s["records"], s["peak_index_exact"], s["near_ties"],
                                                   s["mismatches"], s["accepted_ref"], s["accepted_gpu"]), "",
               "| field | max abs delta (all) | max rel delta (all) | max delta, accepted records |",
               "|---|---|---|---|"]
        for f in self.FIELDS:
            unit = " (samples)" if f in ("subsample_offset", "toa_samples") else ""
            out.append("| %s%s | %.3g | %s | %.3g%s |" % (
                f, unit, s["max_abs_delta"][f],
                "-" if f in ("subsample_offset", "toa_samples") else "%.3g" % s["max_rel_delta"][f],
                s["max_delta_accepted_records"][f], " abs" if f in ("subsample_offset", "toa_samples") else " rel"))
        if self.near_ties:
            out += ["", "Near-ties (peak index differs; margin = (|xc_ref[j_ref]| - |xc_ref[j_gpu]|) / "
                        "|xc_ref[j_ref]| on the reference's own xc):", "",
                    "| code, bin, window_start | j_ref | j_gpu | margin | score_ref | accepted |", "|---|---|---|---|---|---|"]
            for t in self.near_ties:
                out.append("| %s | %d | %d | %.3g | %.4f | %s |" % (t["key"], t["j_ref"], t["j_gpu"], t["margin"],
                                                                 t["score_ref"], t["accepted"]))
        return "\n".join(out) + "\n"

    def json(self):
        return json.dumps(self.summary(), indent=1, default=str)


def compare_detections(got, want, sample_rate, tie_ok=None, rel=REL, xc_ref=None, eps=2e-6, pc_ref=None,
                       report=None, margin_of=None):
    """Return a list of mismatch descriptions (empty = parity).

    got/want are equally long record arrays in the same (code, bin, window)
    order -- a short or reordered result is itself a mismatch.  xc_ref[code]
    (the reference's xc rows) enables the conditioning-aware offset bound;
    pc_ref = (u, {code: replica_d}) the conditioning-aware p_c bound.  A
    differing peak index is accepted only as a documented near-tie: tie_ok(g,
    w) true, or margin_of(g, w) (the margin on the reference's xc) below
    NEAR_TIE; near-ties still need accept/partial exact and w_c, score within
    tolerance (both lags' values differ by less than the margin), and are
    recorded in `report` with their margins."""
    bad = []
    if len(got) != len(want):
        return [("length", len(got), len(want))]
    for g, w in zip(got, want):
        key = (int(w["code_index"]), int(w["bin"]), int(w["window_start"]))
        gkey = (int(g["code_index"]), int(g["bin"]), int(g["window_start"]))
        if gkey != key:
            bad.append((key, "record key", gkey))
            continue
        acc = bool(w["accepted"])
        if report is not None:
            report.records += 1
            report.accepted_ref += int(acc)
            report.accepted_gpu += int(bool(g["accepted"]))
        near_tie = False
        if int(g["peak_index"]) != int(w["peak_index"]):
            margin = None
            ok = False
            if margin_of is not None:
                margin = margin_of(g, w)
                ok = margin is not None and margin < NEAR_TIE
            elif tie_ok is not None:
                ok = bool(tie_ok(g, w))
                if xc_ref is not None:
                    margin = near_tie_margin(xc_ref[int(w["code_index"])], int(w["peak_index"]),
                                             int(g["peak_index"]))
            if not ok:
                bad.append((key, "peak_index", int(g["peak_index"]), int(w["peak_index"]), margin))
                if report is not None:
                    report.mismatches += 1
                continue
            near_tie = True
            if report is not None:
                report.near_ties.append({"key": key, "j_ref": int(w["peak_index"]), "j_gpu": int(g["peak_index"]),
                                         "margin": float(margin) if margin is not None else float("nan"),
                                         "score_ref": float(w["score"]), "accepted": acc})
        elif report is not None:
            report.peak_exact += 1
        if bool(g["accepted"]) != bool(w["accepted"]) or bool(g["partial"]) != bool(w["partial"]):
            bad.append((key, "accept/partial", (g["accepted"], g["partial"]), (w["accepted"], w["partial"])))
        scale = float(np.sqrt(max(float(w["q"]), 0.0) * 1.0))
        for f in ("w_c", "peak_value", "p_c"):
            gv, wv = float(g[f]), float(w[f])
            tol = rel * abs(wv) + 1e-6 * max(abs(wv), scale, 1.0)
            if f == "p_c" and pc_ref is not None:
                tol += eps * pc_scale(pc_ref[1][int(w["code_index"])], pc_ref[0], int(w["peak_index"]))
            if near_tie:
                tol += NEAR_TIE * abs(wv) if f != "p_c" else abs(wv) + scale   # p_c at another lag
            if abs(gv - wv) > tol:
                bad.append((key, f, gv, wv))
            if report is not None and not near_tie:
                report.field(f, gv, wv, acc)
        for f in ("q", "score"):
            gv, wv = float(g[f]), float(w[f])
            tol = rel * abs(wv) + 1e-7 + (NEAR_TIE * abs(wv) if near_tie and f == "score" else 0.0)
            if near_tie and f == "q":
                tol = abs(wv)   # sum of d^2 over another span
            if abs(gv - wv) > tol:
                bad.append((key, f, gv, wv))
            if report is not None and not near_tie:
                report.field(f, gv, wv, acc)
        if near_tie:
            continue   # offset / ToA refer to different peaks
        xr = None if xc_ref is None else xc_ref[int(w["code_index"])]
        sc = abs(float(w["w_c"]) / float(w["score"])) if float(w["score"]) else 0.0
        dtol = delta_tolerance(xr, int(w["peak_index"]), float(w["subsample_offset"]), eps, sc)
        dd = abs(float(g["subsample_offset"]) - float(w["subsample_offset"]))
        dt = abs(float(g["toa_seconds"]) - float(w["toa_seconds"])) * sample_rate
        if report is not None:
            report.field("subsample_offset", g["subsample_offset"], w["subsample_offset"], acc)
            report.field("toa_samples", float(g["toa_seconds"]) * sample_rate, float(w["toa_seconds"]) * sample_rate,
                         acc)
        if dd > dtol:
            bad.append((key, "subsample_offset", float(g["subsample_offset"]), float(w["subsample_offset"]), dtol))
        if dt > dtol + 1e-6:
            bad.append((key, "toa", float(g["toa_seconds"]), float(w["toa_seconds"])))
    return bad


class LazyXc:
    """xc[k] = sum_i dc[i] d[k+i] of the reference's own d and replica d^(c)
    (detector.cpp:92-100, restated as a direct float64 dot product), computed
    only at the lags the checker asks for: the peak and its neighbours (the
    parabola's conditioning) and, for a near-tie, the two competing lags."""

    def __init__(self, d, dc):
        self.d = np.asarray(d, np.float64)
        self.dc = np.asarray(dc, np.float64)

    def __len__(self):
        return self.d.size

    def __getitem__(self, k):
        k = int(k)
        m = min(self.dc.size, self.d.size - k)
        return float(np.dot(self.dc[:m], self.d[k:k + m])) if m > 0 else 0.0


class RefSlots:
    """Reference-side inputs of the checker for one stream: d, u of
    (window start, lo_freq) from oracle/_ref's demodulate_window and each
    code's replica d^(c) from its prepare_code, computed on demand (ctypes
    releases the GIL: prefetch() spreads them over host threads)."""

    def __init__(self, refpy, cfg, bits, iq, window_len, stream_start=0):
        self.ref, self.cfg, self.bits, self.iq = refpy, cfg, bits, iq
        self.W, self.s0 = window_len, stream_start
        self._du = {}
        self._rep = {}

    def _cfg_lo(self, lo):
        import ctypes
        c = type(self.cfg)()
        ctypes.pointer(c)[0] = self.cfg
        c.lo_freq = float(lo)
        return c

    def du(self, start, lo):
        key = (int(start), float(lo))
        if key not in self._du:
            o = int(start) - self.s0
            self._du[key] = self.ref.demodulate_window(self.iq[2 * o:2 * (o + self.W)], int(start),
                                                       self._cfg_lo(lo))
        return self._du[key]

    def replica(self, code):
        code = int(code)
        if code not in self._rep:
            s = self.ref.Session()
            k = s.prepare_code(self.bits[code], self.cfg, self.W, "c%d" % code)
            self._rep[code] = s.code_replica(k)
            s.close()
        return self._rep[code]

    def prefetch(self, slots=(), codes=(), threads=None):
        import os
        from concurrent.futures import ThreadPoolExecutor
        jobs = [(self.du, s) for s in slots if (int(s[0]), float(s[1])) not in self._du] + \
               [(self.replica, (c,)) for c in codes if int(c) not in self._rep]
        with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1) as ex:
            list(ex.map(lambda j: j[0](*j[1]), jobs))

    def compare(self, got, want, start, lo, sample_rate, report=None, code_offset=0, eps=1e-5):
        """compare_detections for the records of one (window, bin) slot, with
        the conditioning-aware offset and p_c bounds and near-tie margins on
        the reference's own d and replicas."""
        d, u = self.du(start, lo)
        codes = sorted({int(c) for c in want["code_index"]})
        reps = {c: self.replica(c - code_offset) for c in codes}
        xc = {c: LazyXc(d, reps[c]) for c in codes}

        def margin_of(g, w):
            return near_tie_margin(xc[int(w["code_index"])], int(w["peak_index"]), int(g["peak_index"]))

        return compare_detections(got, want, sample_rate, xc_ref=xc, pc_ref=(u, reps), eps=eps, report=report,
                                  margin_of=margin_of)
