"""torchrun worker: N-stage pipeline over NCCL (one stage per GPU) in lockstep
with the oracle pipeline of the same P.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mp_pipeline_worker.py [shape]

Every rank drives the same SPMD call sequence and compares the replicated
tree/schedule state with the oracle; the last rank also compares logits.
Exit code 0 = parity green on every rank.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.distributed as dist

from oracle.pipeline import OraclePipeline
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES, reduced
from tests.lockstep import planted_trees, run_lockstep

SEED = 0x5EED01


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    n_layers = None
    if ":" in name:   # "shape:L" -> the same per-layer shapes with L layers
        name, n_layers = name.split(":")[0], int(name.split(":")[1])
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [F.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    shape = SHAPES[name] if n_layers is None else reduced(name, n_layers)
    P = world
    lps = None
    gp = F.Pipeline(shape, n_stages=P, rank=rank, max_ctx=1024, max_seg=16, device=local,
                    nccl_id=obj[0], layers_per_stage=lps)
    gp.fs_load_random_weights(SEED)
    if rank == P - 1:
        gp.enable_logits()
    st = gp.state()
    op = OraclePipeline(shape, SEED, n_stages=P, layers_per_stage=st["layers_per_stage"],
                        max_slots=1024)
    prefix = gen.prefix_tokens(SEED, 40, shape.vocab)
    xo = op.set_prefix(prefix)
    xg = gp.fs_set_prefix(prefix)
    assert xg == xo, (xg, xo)
    l_max = 8
    if name.startswith("7b"):
        planted, n_nodes, depth, tol, l_max = (0, 3, 9, 18, 25, 33, 40), 64, 6, 2e-2, 16
    elif shape.bf16:
        planted, n_nodes, depth, tol = (0, 2, 5, 17, 21, 33), 40, 6, 2e-2
    else:
        planted, n_nodes, depth, tol = (0, 1, 2, 9), 15, 4, 1e-4
    stats = run_lockstep(gp, op, planted_trees(shape, n_nodes, depth, planted, SEED), n_rounds=4,
                         l_max=l_max, tol=tol)
    # KV rows of this rank's layers: compacted draft rows are the oracle's rows
    s = gp.state()
    for l in range(s["layer_begin"], s["layer_end"]):
        for slot in range(s["l_glo"] - 6, s["l_glo"]):
            a = gp.read_kv(l, 0, 0, slot)
            b = op.kv.get(l, 0, 0, slot)
            assert float(abs(a - b).max()) <= (1e-4 if not shape.bf16 else 2 ** -6), (l, slot)
    print(f"rank {rank}/{P} {name}: ok  rows {stats.rows} decisions {stats.decisions} "
          f"committed {len(stats.committed)} max|dlogit| {stats.max_abs:.2e} layers "
          f"{s['layer_begin']}..{s['layer_end']}", flush=True)
    gp.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
