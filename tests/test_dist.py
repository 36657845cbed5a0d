"""Multi-process (world_size 2, gloo, CPU) test of the frame-sharded decode plumbing:
each rank decodes its own global frame shard (the oracle stands in for the GPU
decode here), counters are all-reduced, and the totals equal a single-process
decode of all frames."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import ldpcgen as g


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _decode_counts(code, cfg, f0, nf):
    import oracle
    from paper_cs_0609090_b200.dist import count_errors_host
    llr = cfg.llrs(code, f0, nf).astype(np.int32)
    r = oracle.decode(code, llr, "compact", "int", cfg.max_iter, cfg.early_stop, cfg.offset_raw, cfg.clamp)
    return count_errors_host(oracle.pack_bits(r.bits), r.ok, r.iters), r


def _worker(rank, world, port, per_rank, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_cs_0609090_b200.dist import frame_shard, reduce_counters
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = g.CONFIGS[1]
    code = cfg.code()
    f0, nf = frame_shard(rank, world, per_rank)
    counts, _ = _decode_counts(code, cfg, f0, nf)
    c = torch.tensor(counts, dtype=torch.int64)
    t = torch.tensor([10.0 + rank], dtype=torch.float64)
    reduce_counters(c, t)
    out[rank] = (c.tolist(), float(t.item()))
    dist.destroy_process_group()


def test_shard_ranges():
    from paper_cs_0609090_b200.dist import frame_shard
    assert frame_shard(0, 4, 100) == (0, 100)
    assert frame_shard(3, 4, 100) == (300, 100)
    with pytest.raises(ValueError):
        frame_shard(4, 4, 100)


def test_two_rank_gloo_counters_match_single_process():
    world, per_rank = 2, 12
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, per_rank, out), nprocs=world, join=True, start_method="spawn")
    cfg = g.CONFIGS[1]
    code = cfg.code()
    total, _ = _decode_counts(code, cfg, 0, world * per_rank)
    for r in range(world):
        counts, t = out[r]
        assert counts == total
        assert t == 11.0          # max over ranks


def test_rank_shards_compose_to_the_global_batch():
    """Per-frame outputs do not depend on the number of ranks (global frame ids)."""
    cfg = g.CONFIGS[1]
    code = cfg.code()
    _, whole = _decode_counts(code, cfg, 0, 8)
    _, a = _decode_counts(code, cfg, 0, 4)
    _, b = _decode_counts(code, cfg, 4, 4)
    assert np.array_equal(np.concatenate([a.post, b.post]), whole.post)
    assert np.array_equal(np.concatenate([a.iters, b.iters]), whole.iters)


def _run_bench(args, timeout=240):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return lines[0]


def test_bench_spawns_two_ranks_and_reduces():
    """`bench.py --gpus 2` with no launcher re-executes itself under torch.distributed.run
    (2 ranks, 127.0.0.1 rendezvous); --dist-check drives the bench's own sharding and SUM /
    MAX all-reduce (gloo on CPU, NCCL on GPUs) end to end and checks them on rank 0."""
    line = _run_bench(["--gpus", "2", "--dist-check", "--config", "1", "--frames", "8"])
    assert line["dist_check"] is True and line["n_ranks"] == 2


def test_bench_reference_arm_two_ranks():
    """The reference arm under 2 ranks: rank 0 alone times the oracle and prints one line."""
    line = _run_bench(["--gpus", "2", "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3",
                       "--ref-frames", "4"])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
