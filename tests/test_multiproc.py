"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host path
(paper_2512_09058_b200/shard.py, used by bench.py under torchrun): each rank
generates and solves its own shard of independent instances with no data-path
collective; the timing reduction is a max over ranks; gathering the shards
reproduces the single-process batch bit for bit. The per-rank solver here is
the C oracle (the GPU path is covered by the -m gpu tests; this checks the
sharding / reduction logic around it)."""
import os
import pickle
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, mode):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from pyoracle import Oracle

    from paper_2512_09058_b200 import shard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    if mode == "weak":
        p, start = shard.generate_shard(1, 3, rank, world, per_rank=3, N=16)
    else:
        p, start = shard.generate_shard(0, 5, rank, world, total=5, N=16)
    sol, rc, _ = Oracle().solve_problem(p, 4 if mode == "strong" else 16)
    t = shard.max_over_ranks(10.0 + rank)  # per-rank "device time"
    full = shard.gather_solutions(sol)
    if rank == 0:
        with open(os.path.join(out_dir, f"{mode}.pkl"), "wb") as fh:
            pickle.dump({"t": t, "rc": rc, "u": full.u, "x": full.x, "lam": full.lam,
                         "start": start}, fh)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_two_rank_sharding_matches_single_process(tmp_path, mode):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), mode), nprocs=world, join=True)
    with open(tmp_path / f"{mode}.pkl", "rb") as fh:
        r = pickle.load(fh)
    assert r["t"] == 11.0  # max over ranks
    assert r["rc"] == 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle

    from paper_2512_09058_b200 import synth
    if mode == "weak":
        whole, P = synth.generate(1, seed=3, batch=6, N=16), 16
    else:
        whole, P = synth.generate(0, seed=5, batch=5, N=16), 4
    ref, rc, _ = Oracle().solve_problem(whole, P)
    assert rc == 0
    for k in ("u", "x", "lam"):
        assert np.array_equal(r[k], getattr(ref, k)), k


def test_shard_bounds_cover_exactly():
    from paper_2512_09058_b200.shard import shard_bounds
    for total in (0, 1, 7, 1024):
        for world in (1, 2, 3, 8):
            got = [shard_bounds(total, r, world) for r in range(world)]
            assert sum(c for _, c in got) == total
            pos = 0
            for s, c in got:
                assert s == pos
                pos += c
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


def _gpu_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_2512_09058_b200 import kkt, shard

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    p, start = shard.generate_shard(1, 7, rank, world, total=9, N=32)
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=16), ctx=kkt.Context(rank))
    full = shard.gather_solutions(sol)
    if rank == 0:
        with open(os.path.join(out_dir, "gpu.pkl"), "wb") as fh:
            pickle.dump({"u": full.u, "x": full.x, "lam": full.lam}, fh)
    dist.destroy_process_group()


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_two_gpu_ranks_match_single_gpu(tmp_path):
    # one process per GPU, each solving its strong-scaling shard on its own
    # context (kkt.Context(local_rank)); the gathered batch equals the
    # single-GPU solve of the whole batch bit for bit
    mp.spawn(_gpu_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    with open(tmp_path / "gpu.pkl", "rb") as fh:
        r = pickle.load(fh)
    from paper_2512_09058_b200 import kkt, synth
    whole = synth.generate(1, seed=7, batch=9, N=32)
    ref = kkt.solve_problem(whole, kkt.FactorOptions(P=16))
    for k in ("u", "x", "lam"):
        assert np.array_equal(r[k], getattr(ref, k)), k


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_bench_two_ranks_strong_scaling():
    import json
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", "1", "--extra", "none", "--steps", "2", "--warmup", "3", "--no-cpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900).stdout
    line = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["batch"] == 1024 and line["config"]["batch_per_gpu"] == 512
    assert line["parity"]["ok"]
