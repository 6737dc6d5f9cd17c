"""CPU, world_size 2 over gloo: tag-set sharding + detection gather (the
multi-GPU host path of bench.py), checked against a single-process run.  The
per-rank detections come from the oracle restatement (no GPU here)."""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import oraclepy as O
    from paper_2005_10445_b200 import dist as tdist
    from paper_2005_10445_b200._abi import desk_config
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = np.load(os.path.join(ROOT, "tests", "golden", "desk_e2e.npz"))
    cfg = desk_config(1024)
    W = z["d"].size
    b, e = tdist.shard_codes(len(z["bits"]), rank, world)
    codes = [O.prepare_code(x, cfg, W) for x in z["bits"][b:e]]
    det = O.detect(z["d"], z["u"], codes, 0.25, 0, cfg.mod.sample_rate)
    merged = tdist.gather_detections(det, b)
    if rank == 0:
        q.put(merged.tobytes())
    dist.destroy_process_group()


def test_two_rank_shard_and_gather():
    from paper_2005_10445_b200 import dist as tdist
    from paper_2005_10445_b200._abi import DETECTION_DTYPE
    assert [tdist.shard_codes(10, r, 4) for r in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=300), dtype=DETECTION_DTYPE)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    z = np.load(os.path.join(ROOT, "tests", "golden", "desk_e2e.npz"))
    want = z["det"].view(DETECTION_DTYPE)
    assert got.tobytes() == want.tobytes()
