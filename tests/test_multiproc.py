"""Multi-process host logic on CPU (gloo, world_size 2).

The path shards by utterance with no data-path collective:
each rank renders its LPT shard; the union of the shards must equal the
single-process render byte for byte (outputs do not depend on the parallelism
degree).  The per-rank compute here is the CPU oracle standing in
for the device (there is no GPU in this container); the sharding, timing
reduction and gather logic are the ones bench.py uses.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1712_03439_b200 import scenes, shard

    full = scenes.config3(n_utt=6, seed=77)
    sub, ids = shard.shard_batch(full, rank, world)
    out, out_len, layout, gains, power = oracle.port().render_batch(sub)
    per_utt = {}
    for k, u in enumerate(ids):
        J = int(np.diff(sub.mic_begin)[k])
        per_utt[int(u)] = [sub.channel(out, k, j, out_len[k]).copy() for j in range(J)]
    gathered = [None] * world
    dist.all_gather_object(gathered, per_utt)
    # the optional final gather of the output buffers themselves (shard.gather_outputs)
    got = shard.gather_outputs(torch.from_numpy(np.ascontiguousarray(out)), ids, out_len)
    if rank == 0:
        assert len(got) == world
        for r, (g_ids, g_len, g_out) in enumerate(got):
            sub_r, ids_r = shard.shard_batch(full, r, world)
            assert (g_ids == ids_r).all()
            if r == rank:
                assert (g_len == out_len).all() and (g_out.numpy() == out).all()
            for k, u in enumerate(g_ids):
                J = int(np.diff(sub_r.mic_begin)[k])
                for j in range(J):
                    ch = sub_r.channel(g_out.numpy(), k, j, g_len[k])
                    assert (ch == gathered[r][int(u)][j]).all()
    else:
        assert got is None
    # bench.py's timing reduction: max over ranks
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        merged = {}
        for d in gathered:
            assert not set(d) & set(merged), "an utterance was rendered twice"
            merged.update(d)
        q.put((merged, float(t[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_lpt_partition_properties():
    from paper_1712_03439_b200 import scenes, shard

    b = scenes.config4(n_utt=64, signals=False)
    w = shard.predicted_work(b)
    for world in (1, 2, 4, 8):
        parts = shard.lpt_partition(w, world)
        allids = np.sort(np.concatenate(parts))
        assert (allids == np.arange(b.n_utt)).all()
        loads = np.array([w[p].sum() for p in parts])
        assert loads.max() <= loads.mean() + w.max()  # LPT bound


def test_gloo_two_ranks_match_single_process():
    import oracle
    from paper_1712_03439_b200 import scenes

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax == 2.0
    full = scenes.config3(n_utt=6, seed=77)
    out, out_len, *_ = oracle.port().render_batch(full)
    assert sorted(merged) == list(range(full.n_utt))
    for u in range(full.n_utt):
        for j, ch in enumerate(merged[u]):
            want = full.channel(out, u, j, out_len[u])
            assert (ch.view(np.uint64) == want.view(np.uint64)).all()


def _bench_json(args, env=None):
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, cwd=root, env=e,
                       capture_output=True, text=True, timeout=600)
    return r, [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("scaling,world", [("strong", 2), ("weak", 2), ("strong", 4)])
def test_bench_spawns_ranks_and_covers_the_workload(scaling, world):
    """`python bench.py --gpus N` with WORLD_SIZE unset spawns N ranks (here on CPU with
    gloo, --dry-run): every utterance of the job lands on exactly one rank, the timing
    reduction is the max over ranks, and rank 0 alone prints."""
    r, lines = _bench_json(["--gpus", str(world), "--dry-run", "--scaling", scaling, "--utterances", "256"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == world and d["covers_every_utterance_once"] and d["max_over_ranks"] == float(world)
    assert len(d["shard_utterances"]) == world
    total = 256 * (world if scaling == "weak" else 1)
    assert sum(d["shard_utterances"]) == total == d["config"]["utterances"]
    if scaling == "strong":  # LPT bound: shards within one utterance's predicted work of each other
        a = np.array(d["shard_predicted_work"])
        assert a.max() - a.min() <= d["max_utterance_work"] * (1 + 1e-9)


def test_bench_rejects_gpus_world_mismatch():
    r, _ = _bench_json(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
