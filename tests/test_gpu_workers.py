"""PyTorch workers on the engine: ResNet-20 parameters and
gradients live as views of flat CUDA buffers; push hands the engine the
gradient's device pointer, pull writes the parameters in place. The server's
weights must equal, bit for bit, an fp32 replay of the same pushes
(t = float32(lr) * g rounded, then w - t rounded), and every pull must
deliver exactly the weights current at that moment."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ps = pytest.importorskip("paper_1908_11848_b200")
from paper_1908_11848_b200.workers import CifarResNet, TorchWorker, synthetic_cifar  # noqa: E402


@pytest.mark.parametrize("paradigm,s,r", [("asp", 0, 0), ("dssp", 1, 4), ("bsp", 0, 0)])
def test_resnet20_workers_bit_exact(paradigm, s, r):
    torch.manual_seed(0)
    P = 2
    cfg = ps.validate_config(ps.make_config(paradigm=paradigm, worker_count=P, s_lower=s,
                                            r_max=r, learning_rate=0.01, seed=4))
    workers = [TorchWorker(p, CifarResNet(20), synthetic_cifar(3, 16, seed=p)) for p in range(P)]
    d = workers[0].dimension
    assert d == 272_474
    server = ps.ParameterServer(cfg, d)
    w_ref = torch.from_numpy(ps.initial_weights(cfg, d).values.astype(np.float32)).cuda()
    lr32 = torch.tensor(np.float32(cfg.learning_rate), device="cuda")
    for wk in workers:
        wk.adopt_from(server)
        assert torch.equal(wk.params[:d], w_ref)
    now = 0.0
    pending = set()
    for it in range(12):
        p = it % P
        if p in pending:
            continue
        g = workers[p].begin_iteration()
        gsave = g.values.clone()
        now += 0.5 + p
        dec = server.handle_push(g, now)
        w_ref = w_ref - gsave * lr32
        if dec.granted:
            for q in dec.released:
                pending.discard(q)
                workers[q].adopt_from(server)
                assert torch.equal(workers[q].params[:d], w_ref)
            workers[p].adopt_from(server)
            assert torch.equal(workers[p].params[:d], w_ref)
        else:
            pending.add(p)
    got = torch.from_numpy(np.array(server.weights.values)).cuda()
    assert torch.equal(got.view(torch.int32), w_ref.view(torch.int32))
    assert server.weights.version == sum(w.iterations for w in workers)
