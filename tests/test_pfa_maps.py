"""CPU checks of the prime-factor (Good-Thomas) split the search shape's
correlation runs on (csrc/corr_v3.cuh pfa_split): the
index maps, the Hermitian mirror pass A relies on, the rotated pass-B
epilogue's lag prefix, and -- on small analogues -- the whole two-pass inverse
transform restated in numpy against np.fft.ifft.  No GPU: this pins the
algebra; tests/test_gpu_*.py pin the kernels against the reference."""
import numpy as np
import pytest


def pfa_column_element(k, N1, PA, QA):
    """Storage of spectrum index k: column k1 = k mod N1, element (a, b) with
    a = k mod PA, b = (k mod N1*QA) div N1 (stored at a + PA*b)."""
    return k % N1, k % PA, (k % (N1 * QA)) // N1


def test_search_shape_maps_are_bijections():
    N1, PA, QA = 1024, 27, 32
    N = N1 * PA * QA
    assert N == 884736 and np.gcd(PA, N1 * QA) == 1
    k = np.arange(N, dtype=np.int64)
    k1, a, b = pfa_column_element(k, N1, PA, QA)
    flat = k1 * (PA * QA) + a + PA * b
    assert np.unique(flat).size == N
    # the forward pass stores natural k2 = k div N1 of column k1 at
    # (k2 mod QA) * PA + (k1 + N1 k2) mod PA (kernels.cuh k_fwd_pass2 pos())
    k2 = k // N1
    assert np.array_equal(a + PA * b, (k2 % QA) * PA + (k1 + N1 * k2) % PA)


def test_search_shape_mirror_rule():
    """N - k for k in column cp, element (a, b): column (N1 - cp) mod N1,
    element ((PA - a) mod PA, QA - 1 - b) -- or ((PA - a) mod PA, (QA - b) mod QA)
    in column 0 (corr_v3.cuh item_passA)."""
    N1, PA, QA = 1024, 27, 32
    N = N1 * PA * QA
    rng = np.random.default_rng(1)
    k = rng.integers(1, N, size=200000)
    k1, a, b = pfa_column_element(k, N1, PA, QA)
    m1, ma, mb = pfa_column_element(N - k, N1, PA, QA)
    assert np.array_equal(m1, (N1 - k1) % N1)
    assert np.array_equal(ma, (PA - a) % PA)
    assert np.array_equal(mb, np.where(k1 == 0, (QA - b) % QA, QA - 1 - b))


@pytest.mark.parametrize("W", [800000, 870000, 884736, 700000, 27648, 5])
def test_rotated_epilogue_lags(W):
    """Pass B, column t2 = t_b1 + QA t_a, lane c: base = (N/PA) t_a +
    PA (t_b1 + QA c) mod N = q SE + r; after the w_32^{-a q} rotation slot e
    holds lag r + e SE.  Over all (t2, c, e) every lag in [0, N) appears once,
    and the valid ones (t < W) are exactly the slots e < m = ceil((W - r)/SE)."""
    PA, QA, PB, QB, N1 = 27, 32, 32, 32, 1024
    N = N1 * PA * QA
    SE = N // PB
    t2 = np.arange(PA * QA)
    c = np.arange(QB)
    tb1, ta = t2 % QA, t2 // QA
    base = ((N // PA) * ta[:, None] + PA * (tb1[:, None] + QA * c[None, :])) % N
    q, r = base // SE, base % SE
    lags = r[..., None] + SE * np.arange(PB)[None, None, :]
    assert np.unique(lags).size == N and lags.max() < N
    m = np.where(W > r, np.minimum(PB, (W - r + SE - 1) // SE), 0)
    valid = np.arange(PB)[None, None, :] < m[..., None]
    assert np.array_equal(valid, lags < W)
    if W >= (PB - 4) * SE:
        assert (m >= PB - 4).all()   # the kernel's unmasked fast path


def _ifft_two_pass_pfa(Z, PA, QA, N1, P1, Q1):
    """The search-shape inverse transform restated: Z in PFA storage
    [k1][a][b]; pass A per column k1: DFT_QA over b, DFT_PA over a (no
    twiddle between them), times w_{N/PA}^{k1 t_b1}; pass B per (t_a, t_b1):
    DFT_{N1} over k1 (as P1 x Q1 four-step with its own twiddles); output
    (t_a, t_b) is the lag (N/PA t_a + PA t_b) mod N, t_b = t_b1 + QA t_b2."""
    N = N1 * PA * QA
    NB = N // PA
    k = np.arange(N)
    k1, a, b = pfa_column_element(k, N1, PA, QA)
    cols = np.zeros((N1, PA, QA), complex)
    cols[k1, a, b] = Z
    # pass A (inverse: + sign)
    y = np.fft.ifft(cols, axis=2) * QA          # over b -> t_b1
    y = np.fft.ifft(y, axis=1) * PA             # over a -> t_a
    tb1 = np.arange(QA)
    y *= np.exp(2j * np.pi * np.outer(np.arange(N1), tb1) / NB)[:, None, :]
    # pass B over k1 (four-step P1 x Q1 restated as one DFT of length N1)
    z = np.fft.ifft(y, axis=0) * N1             # -> t_b2
    out = np.zeros(N, complex)
    tb2 = np.arange(N1)
    ta = np.arange(PA)
    t_b = tb1[None, None, :] + QA * tb2[:, None, None]
    lag = ((N // PA) * ta[None, :, None] + PA * t_b) % N
    out[lag] = z
    return out


@pytest.mark.parametrize("PA,QA,N1", [(3, 4, 8), (5, 8, 16), (27, 32, 16)])
def test_two_pass_pfa_inverse_equals_ifft(PA, QA, N1):
    N = N1 * PA * QA
    assert np.gcd(PA, N1 * QA) == 1
    rng = np.random.default_rng(PA * 1000 + N1)
    Z = rng.normal(size=N) + 1j * rng.normal(size=N)
    got = _ifft_two_pass_pfa(Z, PA, QA, N1, None, None)
    want = np.fft.ifft(Z) * N
    assert np.abs(got - want).max() <= 1e-9 * np.abs(want).max()


def test_segmented_lag_ranges_cover_window():
    """Segmented correlation (tagdsp_gpu.cu seg_lags): segments g of B =
    2^20 - n + 1 lags cover [0, W) exactly once, each from at most
    B + n - 1 <= 2^20 samples (no wrap-around)."""
    Nmax = 1 << 20
    for W, n in [(1200000, 65741), (2000000, 65741), (982836, 65741), (1048577, 1)]:
        B = Nmax - n + 1
        nseg = (W + B - 1) // B
        covered = np.zeros(W, np.int32)
        for g in range(nseg):
            o = g * B
            lag_lim = min(B, W - o)
            data = min(W - o, B + n - 1)
            assert lag_lim + n - 1 <= Nmax and data <= Nmax
            covered[o:o + lag_lim] += 1
        assert (covered == 1).all()


def test_output_rotation_identity():
    """The pass-B rotation: taking the step-2 twiddle as w_1024^{a (c - 32 q)}
    = w_1024^{a c} w_32^{-a q} makes the last DFT_32's slot e hold output
    e - q (mod 32) -- i.e. lag r + e SE instead of (q SE + r + e SE) mod N."""
    rng = np.random.default_rng(7)
    P = 32
    x = rng.normal(size=P) + 1j * rng.normal(size=P)
    Y = np.fft.ifft(x) * P                      # sum_a x[a] w^{+a e}
    for q in range(P):
        xr = x * np.exp(-2j * np.pi * np.arange(P) * q / P)
        Yr = np.fft.ifft(xr) * P
        assert np.allclose(Yr, np.roll(Y, q), atol=1e-9)
        # anchors a = 8j: w_1024^{-256 j q} = i^{-j q}
        for j in (1, 2, 3):
            assert np.isclose(np.exp(-2j * np.pi * 256 * j * q / 1024), 1j ** ((4 - j) * q % 4))
