"""N>1 host path on CPU: world_size-2 gloo processes run the handshake bench.py uses for
one-process-per-GPU runs — NCCL id broadcast, every rank deriving the identical rule plan
independently, dp batch slicing, and max-over-ranks timing."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2310_16355_b200 import dist as D
    from paper_2310_16355_b200 import rules

    info = D.rank_info()
    dist = D.init_host_group(info)
    nccl_id = D.share_nccl_id(dist, info.rank)
    spec = rules.read_model_spec(os.path.join(ROOT, "oracle", "specs", "llama7b_vocab_parallel.spec"))
    plan = rules.derive_plan(rules.transformer_param_shapes(spec), world, spec.overrides)
    plans = [None] * world
    dist.all_gather_object(plans, plan.serialize())
    ids = [None] * world
    dist.all_gather_object(ids, nccl_id)
    t = D.max_over_ranks(dist, float(rank + 1) * 1.5)
    batch = np.arange(4 * 8).reshape(4, 8)
    mine = D.replica_rows(batch, world, rank)
    slices = [None] * world
    dist.all_gather_object(slices, mine.tolist())
    out.put((rank, len(set(plans)), len(set(ids)), len(nccl_id), t, slices))
    dist.destroy_process_group()


def test_two_rank_handshake():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, n_plans, n_ids, id_len, t, slices in res:
        assert n_plans == 1  # every rank derived the same plan
        assert n_ids == 1 and id_len == 128  # one NCCL id, broadcast from rank 0
        assert t == 3.0  # max over ranks
        assert np.concatenate([np.array(s) for s in slices]).tolist() == np.arange(32).reshape(4, 8).tolist()


def test_mesh_coords_match_reference_layout():
    from paper_2310_16355_b200 import dist as D

    # mesh.hpp:25-34 / mesh.cpp:7-17 for the cfg3 2 x 4 mesh
    assert D.mp_group(1, 4) == [4, 5, 6, 7]
    assert D.dp_group(2, 2, 4) == [2, 6]
    assert [D.mesh_coords(d, 2, 4) for d in (0, 5, 7)] == [(0, 0), (1, 1), (1, 3)]
