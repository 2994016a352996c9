"""One rank of the PyTorch-workers-on-the-sharded-server check (launched by
tests/test_gpu_sharded.py under torchrun).

Every rank trains a CIFAR ResNet-20 whose parameters live IN the server's
replica and whose gradients live IN the server's update buffer (no copies):
backward writes the push, a run of the sharded server applies every worker's
update in ticket order and writes the new weights straight into every
replica. After each step rank 0 checks its replica bit for bit against an
fp32 replay of the all-gathered gradients in the ticket order the REFERENCE
simulator produces for this schedule (tests/golden/c3_schedule.json.gz;
server.py:37; simnet.py:167-201), and the device gate's trace against the
same reference rows."""

import json
import os
import sys

import torch
import torch.distributed as dist
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1908_11848_b200 as ps  # noqa: E402
from paper_1908_11848_b200.sharded import ShardedServer, homogeneous_push_times  # noqa: E402
from paper_1908_11848_b200.workers import CifarResNet, flatten_, synthetic_cifar  # noqa: E402


def main(out_dir):
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    checks = []
    for paradigm, s, r in (("asp", 0, 0), ("dssp", 3, 12)):
        torch.manual_seed(0)  # identical initial weights on every rank
        model = CifarResNet(20).cuda()
        w0 = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
        d = w0.numel()
        lr = 0.01
        cfg = ps.validate_config(ps.make_config(paradigm=paradigm, worker_count=world, s_lower=s, r_max=r,
                                                learning_rate=lr, seed=0, dimension=d))
        srv = ShardedServer(cfg, d, rank, world, local, w0_device=w0)
        flatten_(model, into=(srv.replica, srv.update), copy_params=False)
        assert torch.equal(srv.replica[:d], w0)
        batches = synthetic_cifar(4, 32, seed=100 + rank)
        times = homogeneous_push_times(1.0, 0.05, 8)
        w_ref = w0.clone()
        lr32 = torch.tensor(lr, dtype=torch.float32, device="cuda")
        ok = True
        ref = next(x for x in oracle.load_golden("c3_schedule.json.gz")["runs"]
                   if x["name"] == f"c3_{paradigm}_p{world}")
        ref_rows = [ln.split("\t") for ln in ref["trace"].splitlines() if ln.split("\t")[2] == "push_arrive"]
        for step in range(6):
            x, y = batches[step % len(batches)]
            srv.update.zero_()
            loss = F.cross_entropy(model(x), y)
            loss.backward()
            grads = [torch.empty(d, device="cuda") for _ in range(world)]
            dist.all_gather(grads, srv.update[:d].contiguous())
            srv.run(times[step:step + 1])
            # this group's ticket order as the reference serves it
            order = [int(row[1]) for row in ref_rows[step * world:(step + 1) * world]]
            got = [e.render().split("\t") for e in srv.trace()][-world:]
            ok = ok and got == ref_rows[step * world:(step + 1) * world]
            for q in order:
                w_ref = w_ref - grads[q] * lr32
            ok = ok and bool(torch.equal(srv.replica[:d].view(torch.int32), w_ref.view(torch.int32)))
        checks.append({"paradigm": paradigm, "ok": ok, "version": int(srv.state().version),
                       "loss": float(loss)})
        torch.cuda.synchronize()
        dist.barrier()
        srv.close()
    with open(os.path.join(out_dir, f"torch_rank{rank}.json"), "w") as fh:
        json.dump(checks, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
