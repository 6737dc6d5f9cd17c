"""Two ranks on one B200 over gloo: tag-set sharding + detection gather on
the real GPU path (tdg_search per rank on its roster slice), checked bitwise
against a single-rank search of the whole roster.  The multi-GPU layout of
bench.py (north star: "shards naturally ... by tag set, with only the detection
lists gathered at the end") with both ranks sharing cuda:0."""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

W = 12000
ADV = 10000
N_WIN = 3
BINS = np.array([-100e3, 0.0, 100e3])
N_CODES = 7   # odd: rank 0 gets 4 codes (2 pairs), rank 1 gets 3 (a half-empty pair)


def _scene():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy
    from paper_2005_10445_b200._abi import desk_config
    cfg = desk_config(1024)
    bits = np.stack([refpy.gen_code(200 + i, cfg) for i in range(N_CODES)])
    n = ADV * (N_WIN - 1) + W
    # two codes in the stream, one in each rank's slice (window 0 and window 2)
    a = refpy.channel_window(bits[1], cfg, 1234.25, n, 77, snr_db=12.0).astype(np.int32)
    b = refpy.channel_window(bits[5], cfg, 21000.5, n, 78, snr_db=12.0).astype(np.int32)
    iq = np.clip(a + b, -32767, 32767).astype(np.int16)
    return cfg, bits, iq


def _search(dev, cfg, bits, iq):
    from paper_2005_10445_b200 import capi
    ctx = capi.Context(dev)
    cs = capi.CodeSet.prepare(ctx, cfg, W, bits)
    recs = capi.search(ctx, cfg, BINS, iq, cs, W, ADV)
    return recs


def _worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2005_10445_b200 import dist as tdist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, bits, iq = _scene()
    b, e = tdist.shard_codes(N_CODES, rank, world)
    recs = _search(0, cfg, bits[b:e], iq)
    merged = tdist.gather_detections(recs.reshape(-1), b)
    if rank == 0:
        q.put(merged.tobytes())
    dist.destroy_process_group()


def test_two_ranks_one_gpu_match_single_rank():
    from paper_2005_10445_b200 import dist as tdist
    from paper_2005_10445_b200._abi import DETECTION_DTYPE
    sys.path.insert(0, ROOT)
    cfg, bits, iq = _scene()
    single = _search(0, cfg, bits, iq).reshape(-1)
    # single-rank records in the gathered order (window_start, bin, code_index)
    order = np.lexsort((single["code_index"], single["bin"], single["window_start"]))
    rows = single.view(np.uint8).reshape(-1, DETECTION_DTYPE.itemsize)
    want = np.ascontiguousarray(rows[order]).view(DETECTION_DTYPE).reshape(-1)
    acc = want[want["accepted"] == 1]
    assert {1, 5} <= set(acc["code_index"].tolist())   # both injected codes found
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=600), dtype=DETECTION_DTYPE)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(got) == len(want) == N_CODES * N_WIN * len(BINS)
    assert got.tobytes() == want.tobytes()
    assert tdist.shard_codes(N_CODES, 1, 2) == (4, 7)
