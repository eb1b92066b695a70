"""Utterance sharding across GPUs.

Utterances share nothing, so the path shards with no
collective: every rank renders its own utterances.  Strong scaling uses an
LPT (largest-first) assignment by predicted work; weak scaling gives every
rank its own block of utterance ids.  Both are pure functions of the inputs,
so every rank computes the same assignment without communication.
"""
from __future__ import annotations

import heapq

import numpy as np


def predicted_work(batch) -> np.ndarray:
    """Per-utterance device time proxy, known before any RIR is synthesized:
    I * J * (N_x + 0.65 (2K + 1)^3).  The OLA filter costs ~20 N_x log2 N flops per pair
    with log2 N ~ 10 at config 4 (the truncated N_h is not known yet; its log barely
    moves the cost), the image-method synthesis ~(2K + 1)^3 images per pair; the 0.65
    weight is their measured ratio on B200 (config 4: K4 27 ms for 1.05e12 flops, K1
    5.8 ms for 2.1e9 images)."""
    I = np.diff(batch.src_begin)
    J = np.diff(batch.mic_begin)
    nx = batch.sig_len[batch.src_begin[:-1]].astype(np.float64)
    images = (2.0 * batch.image_order.astype(np.float64) + 1.0) ** 3
    return I * J * (nx + 0.65 * images)


def lpt_partition(work: np.ndarray, world: int) -> list:
    """Largest-processing-time-first: returns `world` sorted index arrays."""
    order = np.argsort(-work, kind="stable")
    heap = [(0.0, r) for r in range(world)]
    parts = [[] for _ in range(world)]
    for u in order:
        load, r = heapq.heappop(heap)
        parts[r].append(int(u))
        heapq.heappush(heap, (load + float(work[u]), r))
    return [np.array(sorted(p), dtype=np.int64) for p in parts]


def shard_batch(batch, rank: int, world: int):
    """The sub-batch rank `rank` renders under strong scaling."""
    if world <= 1:
        return batch, np.arange(batch.n_utt)
    part = lpt_partition(predicted_work(batch), world)[rank]
    return batch.subset(part), part


def gather_outputs(out, ids, out_len, dst: int = 0):
    """The optional final gather (north star: "NCCL only for an optional final gather"): every
    rank's mixed output buffer, its utterance ids and output lengths to rank `dst`, over the
    process group's backend (NCCL on GPUs: device-to-device over NVLink; gloo on CPU).  Not on
    the render path — ranks share nothing until here.

    out: this rank's 1-D float32 tensor (device or CPU); ids / out_len: 1-D int64 arrays.
    Returns on `dst` a list of (ids, out_len, out) per rank, `out` trimmed to the rank's size;
    None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    ids_t = torch.as_tensor(np.asarray(ids, np.int64))
    len_t = torch.as_tensor(np.asarray(out_len, np.int64))
    if world == 1:
        return [(ids_t.numpy(), len_t.numpy(), out)]
    rank = dist.get_rank()
    dev = out.device
    # sizes first (buffers are padded to the largest: gather needs equal shapes)
    sizes = torch.tensor([out.numel(), ids_t.numel()], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    n_out = int(max(int(s[0]) for s in all_sizes))
    n_ids = int(max(int(s[1]) for s in all_sizes))
    pad_out = torch.zeros(n_out, dtype=out.dtype, device=dev)
    pad_out[: out.numel()] = out
    meta = torch.zeros(2 * n_ids, dtype=torch.int64, device=dev)
    meta[: ids_t.numel()] = ids_t.to(dev)
    meta[n_ids: n_ids + len_t.numel()] = len_t.to(dev)
    outs = [torch.empty_like(pad_out) for _ in range(world)] if rank == dst else None
    metas = [torch.empty_like(meta) for _ in range(world)] if rank == dst else None
    dist.gather(pad_out, outs, dst=dst)
    dist.gather(meta, metas, dst=dst)
    if rank != dst:
        return None
    res = []
    for r in range(world):
        no, ni = int(all_sizes[r][0]), int(all_sizes[r][1])
        res.append((metas[r][:ni].cpu().numpy(), metas[r][n_ids: n_ids + ni].cpu().numpy(), outs[r][:no]))
    return res
