"""P>1 bench diagnostic: AR greedy stream vs tree acceptance round by round."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
import bench
rank = int(os.environ["RANK"]); P = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
obj = [F.nccl_unique_id() if rank == 0 else None]; dist.broadcast_object_list(obj, src=0)
shape = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "7b"]
ranks = (0, 3, 9, 18, 25, 33, 40)
gp = F.Pipeline(shape, n_stages=P, rank=rank, max_ctx=2048, max_seg=16, device=rank, nccl_id=obj[0])
gp.fs_load_random_weights(bench.SEED)
prefix = gen.prefix_tokens(bench.SEED, 1024, shape.vocab)
x0 = gp.fs_set_prefix(prefix)
stream = bench.greedy_stream(gp, 6 * 7 + 8)
gp.fs_set_prefix(prefix)
for r in range(6):
    t = gen.planted_tree(bench.SEED + r, 64, 6, stream[r * 7: r * 7 + 8], ranks, shape.vocab)
    if gp.state()["x_new"] != int(t["token"][0]):
        if rank == 0: print("round", r, "root mismatch", gp.state()["x_new"], t["token"][0])
        break
    gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], 16)
    got = []
    while True:
        o = gp.fs_verify_step()
        d = gp.fs_accept()
        if not d.progress: continue
        got += list(d.acc_tokens[:d.n_acc])
        flagged = list(d.flagged_ids[:d.n_flagged])
        gp.fs_prune_and_compact(d)
        if not d.cont: break
    if rank == 0:
        print("round", r, "committed", got, "planned", stream[r*7:r*7+7], "x_new", gp.state()["x_new"], "next", stream[r*7+7], "flagged", flagged)
dist.barrier()
