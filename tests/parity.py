"""Parity helpers: compare B200 detections with the reference's, with the
tolerances the north star states (BASELINE.json): peak index and
accept/partial exact except documented near-ties; ToA, score and
correlation magnitudes within ~1e-4 relative."""
import numpy as np

REL = 1e-4


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


def compare_detections(got, want, sample_rate, tie_ok=None, rel=REL, xc_ref=None, eps=2e-6, pc_ref=None):
    """Return a list of mismatch descriptions (empty = parity).  xc_ref[code]
    (the reference's xc rows) enables the conditioning-aware offset bound;
    pc_ref = (u, {code: replica_d}) the conditioning-aware p_c bound."""
    bad = []
    for g, w in zip(got, want):
        key = (int(w["code_index"]), int(w["bin"]), int(w["window_start"]))
        if int(g["peak_index"]) != int(w["peak_index"]):
            if tie_ok is not None and tie_ok(g, w):
                continue
            bad.append((key, "peak_index", int(g["peak_index"]), int(w["peak_index"])))
            continue
        if bool(g["accepted"]) != bool(w["accepted"]) or bool(g["partial"]) != bool(w["partial"]):
            bad.append((key, "accept/partial", (g["accepted"], g["partial"]), (w["accepted"], w["partial"])))
        scale = float(np.sqrt(max(float(w["q"]), 0.0) * 1.0))
        for f in ("w_c", "peak_value", "p_c"):
            gv, wv = float(g[f]), float(w[f])
            tol = rel * abs(wv) + 1e-6 * max(abs(wv), scale, 1.0)
            if f == "p_c" and pc_ref is not None:
                tol += eps * pc_scale(pc_ref[1][int(w["code_index"])], pc_ref[0], int(w["peak_index"]))
            if abs(gv - wv) > tol:
                bad.append((key, f, gv, wv))
        for f in ("q", "score"):
            gv, wv = float(g[f]), float(w[f])
            if abs(gv - wv) > rel * abs(wv) + 1e-7:
                bad.append((key, f, gv, wv))
        xr = None if xc_ref is None else xc_ref[int(w["code_index"])]
        sc = abs(float(w["w_c"]) / float(w["score"])) if float(w["score"]) else 0.0
        dtol = delta_tolerance(xr, int(w["peak_index"]), float(w["subsample_offset"]), eps, sc)
        if abs(float(g["subsample_offset"]) - float(w["subsample_offset"])) > dtol:
            bad.append((key, "subsample_offset", float(g["subsample_offset"]), float(w["subsample_offset"]), dtol))
        if abs(float(g["toa_seconds"]) - float(w["toa_seconds"])) * sample_rate > dtol + 1e-6:
            bad.append((key, "toa", float(g["toa_seconds"]), float(w["toa_seconds"])))
    return bad
