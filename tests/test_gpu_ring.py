"""Device-resident CircularBuffer (tdg_ring_*) on the GPU: push / read / gap /
eviction semantics against the reference's CircularBuffer compiled in place
(oracle/_ref, proj/src/scheduler.cpp:7-45), and searches /
tracking tasks that read their windows from the ring against the same passes
over a linear block (identical kernels, so identical records)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class RefRing:
    """The reference's CircularBuffer compiled in place (oracle/_ref,
    proj/src/scheduler.cpp:7-45) behind the interface the test uses."""

    def __init__(self, ref, cap):
        self.r = ref.Ring(cap)

    def push(self, iq, start):
        return self.r.push(iq, start)

    def read(self, start, end):
        return self.r.read(start, end)

    @property
    def head(self):
        return self.r.bounds()[0]

    @property
    def tail(self):
        return self.r.bounds()[1]


def test_ring_semantics_match_reference(gpu_ctx, ref):
    from paper_2005_10445_b200 import capi
    rng = np.random.default_rng(3)
    cap = 1000
    ring, ref = capi.Ring(gpu_ctx, cap), RefRing(ref, cap)
    t = 0
    # contiguous pushes (wrap-around and eviction), a gap, a block larger than
    # the capacity, an empty block
    plan = [(300, None), (450, None), (400, None), (999, None), (10, 5000), (2500, None), (0, None), (1, None)]
    for n, jump in plan:
        start = jump if jump is not None else t
        blk = rng.integers(-30000, 30000, 2 * n, dtype=np.int16)
        assert ring.push(blk, start) == ref.push(blk, start)
        t = start + n
        assert (ring.head, ring.tail) == (ref.head, ref.tail)
        for a, b in [(ref.head, ref.tail), (ref.tail - 37, ref.tail), (ref.head, ref.head + 500),
                     (ref.head - 1, ref.tail), (ref.head, ref.tail + 1), (ref.tail, ref.tail)]:
            got, want = ring.read(a, b), ref.read(a, b)
            if want is None:
                assert got is None, (a, b)
            else:
                assert got is not None and np.array_equal(got, want), (a, b)


def test_search_and_track_from_ring_match_linear(gpu_ctx, ref):
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import desk_config
    cfg = desk_config(1024)
    P = 1024 * 8
    W = P + 3000
    adv = 2500
    seeds = [300, 301, 302]
    bits = np.stack([ref.gen_code(s, cfg) for s in seeds])
    inj = [(0, 0.004, 1.0, 0.0), (2, 0.0131, 0.7, 2.0e3)]
    iq = ref.generate_recording(cfg, seeds, 0.03, 10.0, 9, inj)
    n = iq.size // 2
    base = 12345                                   # absolute index of the block's first sample
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    bins = [-2.0e3, 0.0, 2.0e3]
    # ring smaller than the stream: windows wrap around its end
    ring = capi.Ring(gpu_ctx, 2 * W + 777)
    pos = 0
    sizes = [7001, 1, 5000, 12000]
    k = 0
    while pos < n:
        m = min(sizes[k % len(sizes)], n - pos)
        ring.push(iq[2 * pos:2 * (pos + m)], base + pos)
        pos += m
        k += 1
    head, tail, _ = ring.bounds()
    first = head + 10
    nw = (tail - first - W) // adv + 1
    assert nw >= 2
    got = capi.search_ring(gpu_ctx, ring, cfg, bins, first, nw, cs, adv)
    lin = iq[2 * (first - base):2 * (first - base + (nw - 1) * adv + W)]
    want = capi.search(gpu_ctx, cfg, bins, lin, cs, W, adv, stream_start=first)
    assert got.tobytes() == want.tobytes()
    starts = [first, first + 777, tail - W, first + adv]
    codes = [0, 2, 1, 1]
    got_t = capi.track_ring(gpu_ctx, ring, cfg, starts, codes, cs)
    want_t = capi.track(gpu_ctx, cfg, iq[2 * (head - base):], starts, codes, cs, stream_start=head)
    assert got_t.tobytes() == want_t.tobytes()
    # windows outside [head, tail) are precondition errors
    with pytest.raises(capi.InvalidArgument):
        capi.search_ring(gpu_ctx, ring, cfg, bins, head - 1, 1, cs, adv)
    with pytest.raises(capi.InvalidArgument):
        capi.track_ring(gpu_ctx, ring, cfg, [tail - W + 1], [0], cs)
