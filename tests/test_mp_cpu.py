"""world_size-2 gloo test of the N>1 SPMD protocol on CPU: each process runs one
pipeline stage (its layer block), hidden rows move by send/recv, the last
stage broadcasts per-row (argmax, margin), every replica runs accept/prune.
The committed stream must equal the single-process P=2 oracle run and greedy
autoregressive decoding (R-def-2)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

SEED = 0x5EED01


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle.pipeline import OraclePipeline
    from synth import gen
    from synth.configs import SHAPES
    from tests.test_oracle_decoder import _run_rounds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = SHAPES["tiny"]
    # trees from the single-process reference (identical on both ranks)
    ref, trees, _ = _run_rounds(shape, 2, 8, 4)
    op = OraclePipeline(shape, SEED, n_stages=world, max_slots=512, rank=rank)
    op.set_prefix(gen.prefix_tokens(SEED, 32, shape.vocab))
    committed = []
    for t in trees:
        op.submit(True, t["parent"], t["token"], t["own"], l_max=8)
        while True:
            op.verify_step()
            d = op.accept()
            if not d["progress"]:
                continue
            committed += d["acc_tokens"]
            op.prune(dict(acc_ids=d["acc_ids"], x_new=d["x_new"], n_new_id=d["n_new_id"],
                          cont=d["cont"]))
            if not d["cont"]:
                break
    q.put((rank, committed, ref, op.snapshot()["l_glo"]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_gloo_pipeline_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, c0, ref0, l0), (r1, c1, ref1, l1) = sorted(res)
    assert c0 == c1 == ref0 and len(c0) == 16 and l0 == l1
