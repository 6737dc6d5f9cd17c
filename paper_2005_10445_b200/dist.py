"""Multi-GPU host plumbing: tag-set sharding and the detection gather.

The acquisition path shards without any data-path exchange: every
(code, window, bin) correlation is independent (batch == sequential bitwise,
proj/tests/acceptance.cpp:153-156), so rank r of R owns a contiguous slice of
the roster and searches the whole stream.  The only collective is the
gather of the per-rank Detection lists at the end of each searched block
(north star: "only the detection lists gathered at the end"), done with
torch.distributed (NCCL on the GPU box, gloo in the CPU tests).
"""
import numpy as np

from ._abi import DETECTION_DTYPE


def shard_codes(n_codes, rank, world):
    """Contiguous [begin, end) slice of the roster owned by `rank`."""
    base, extra = divmod(n_codes, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def gather_detections(records, code_offset, device=None, accepted_only=False):
    """All-gather Detection records from every rank.

    records: DETECTION_DTYPE array with shard-local code_index; code_offset is
    this rank's shard begin (added so indices are roster-global).  Returns the
    merged array on every rank, ordered (window_start, bin, code_index)."""
    import torch
    import torch.distributed as dist

    rows = np.ascontiguousarray(np.asarray(records, dtype=DETECTION_DTYPE)).view(np.uint8).reshape(
        -1, DETECTION_DTYPE.itemsize)
    if accepted_only:
        rows = rows[rows.view(DETECTION_DTYPE).reshape(-1)["accepted"] == 1]
    rows = rows.copy()
    rec = rows.view(DETECTION_DTYPE).reshape(-1)
    rec["code_index"] += np.int32(code_offset)
    raw = torch.from_numpy(rec.view(np.uint8).reshape(-1).copy())
    world = dist.get_world_size()
    n = torch.tensor([raw.numel()], dtype=torch.int64)
    if device is not None:
        n = n.to(device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 1)
    buf = torch.zeros(cap, dtype=torch.uint8)
    buf[:raw.numel()] = raw
    if device is not None:
        buf = buf.to(device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    raw_all = b"".join(o[:s].cpu().numpy().tobytes() for o, s in zip(outs, sizes))
    rows = np.frombuffer(raw_all, dtype=np.uint8).reshape(-1, DETECTION_DTYPE.itemsize)
    merged = rows.view(DETECTION_DTYPE).reshape(-1)
    order = np.lexsort((merged["code_index"], merged["bin"], merged["window_start"]))
    # reorder whole 64-byte rows (structured fancy indexing drops padding bytes)
    return np.ascontiguousarray(rows[order]).view(DETECTION_DTYPE).reshape(-1)
