"""Free-running workers gated by device flags (north star (4); the threaded
runner's loop, runner.py:168-291, with the host out of the iteration loop).

Every worker is a CUDA stream whose iteration -- forward/backward, push
kernel, stream wait on its go flag, pull kernel -- is captured once as a
graph; the host enqueues all iterations up front and synchronizes once.
Parity: the decisions, fed to the CPU oracle gate in the order and at the
device-clock instants the device gate saw them, must come out identical; the
weights must equal the fp32 replay of the pushed updates in ticket order; every
worker's parameters must equal the weights at the version its last pull
recorded."""

import os

import numpy as np
import pytest

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ps = pytest.importorskip("paper_1908_11848_b200")
from paper_1908_11848_b200.engine import Engine  # noqa: E402
from paper_1908_11848_b200.freerun import FreeRunningCluster  # noqa: E402
from paper_1908_11848_b200.workers import SyntheticWorker  # noqa: E402

PARADIGMS = (("dssp", 3, 12), ("ssp", 3, 0), ("bsp", 0, 0), ("asp", 0, 0))


def _check_gate(rep, paradigm, P, s, r):
    gate = oracle.CGate(paradigm, P, s, r)
    for w, now, outcome, released in rep.decision_sequence():
        assert gate.on_push(w, now) == (outcome, released), (w, now)


def _replay(rep, rings, d, w0, lr):
    """fp32 replay of every push in ticket order; returns final weights and
    {version: weights} for the versions the pulls recorded."""
    want_versions = {int(v) for v in rep.pulls["version"]}
    w = w0.copy()
    snaps = {0: w.copy()} if 0 in want_versions else {}
    k = {}
    version = 0
    for row in rep.decisions:
        p = int(row["worker"])
        i = k.get(p, 0)
        k[p] = i + 1
        g = rings[p][i % rings[p].shape[0], :d]
        if row["applied"]:
            w = oracle.apply_f32(w, g, lr)
            version += 1
            assert version == int(row["version"])
            if version in want_versions:
                snaps[version] = w.copy()
    return w, snaps


def _synthetic_cluster(paradigm, s, r, P, d, K, throttle_us, graphs=True, seed=9, devices=None):
    rings_h = []
    for p in range(P):
        ring = np.zeros((K, (d + 3) // 4 * 4), dtype=np.float32)
        for k in range(K):
            ring[k, :d] = oracle.synthetic_update(seed, p, k, d)
        rings_h.append(ring)
    devices = devices or [0] * P
    workers = [SyntheticWorker(torch.from_numpy(rg).to(f"cuda:{devices[p]}"), device=f"cuda:{devices[p]}")
               for p, rg in enumerate(rings_h)]
    eng = Engine(paradigm, P, s, r, 0.05, d, w0=oracle.initial_weights_f64(0, d))
    cl = FreeRunningCluster(eng, workers, throttle_ns=[int(t * 1000) for t in throttle_us],
                            graphs=graphs)
    cl.capture(warmup=0)
    # capture ran no iteration; every worker's ring index is back at 0
    for wk in workers:
        wk.idx.zero_()
    cl._sync_all()
    return eng, cl, workers, rings_h


@pytest.mark.parametrize("paradigm,s,r", PARADIGMS)
@pytest.mark.parametrize("graphs", [True, False])
def test_free_running_synthetic_workers(paradigm, s, r, graphs):
    P, d, K, iters = 4, 70_001, 3, 40
    # heterogeneous cluster: two fast workers, one 3x and one 6x slower
    throttle_us = [0, 0, 40, 100]
    eng, cl, workers, rings = _synthetic_cluster(paradigm, s, r, P, d, K, throttle_us, graphs)
    rep = cl.run(iters)
    assert rep.pushes == P * iters and rep.pulls.size == P * iters
    assert all(rep.iterations[p] == iters for p in range(P))
    _check_gate(rep, paradigm, P, s, r)
    w0 = oracle.initial_weights_f64(0, d).astype(np.float32)
    w, snaps = _replay(rep, rings, d, w0, 0.05)
    got, version = eng.read()
    assert version == P * iters
    assert np.array_equal(got.view(np.uint32), w.view(np.uint32))
    # every worker's parameters are the snapshot of its last pull
    for p in range(P):
        last = rep.pulls[rep.pulls["worker"] == p][-1]
        mine = workers[p].params[:d].cpu().numpy()
        assert np.array_equal(mine.view(np.uint32), snaps[int(last["version"])].view(np.uint32)), p
    # tickets interleave pushes and pulls in one total order
    tickets = np.sort(np.concatenate([rep.decisions["ticket"], rep.pulls["ticket"]]))
    assert np.array_equal(tickets, np.arange(2 * P * iters, dtype=np.uint64))
    if paradigm in ("bsp", "ssp") and graphs:
        # the 6x worker holds the fast ones back (eagerly, the host's own
        # enqueue rate can keep the workers in step)
        assert rep.defers() > 0
    if paradigm == "asp":
        assert rep.defers() == 0
    eng.close()


@pytest.mark.parametrize("paradigm,s,r", PARADIGMS)
def test_free_running_workers_on_peer_gpus(paradigm, s, r):
    """Workers on every GPU of the box, the server on GPU 0: push / pull
    kernels on the worker's GPU reach the weights, gate and tickets over
    NVLink; go flags are raised remotely. Same parity as on one GPU."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    P, d, K, iters = 4, 70_001, 3, 30
    devices = [p % n for p in range(P)]
    eng, cl, workers, rings = _synthetic_cluster(paradigm, s, r, P, d, K, [0, 20, 60, 120],
                                                 devices=devices)
    rep = cl.run(iters)
    assert rep.pushes == P * iters
    _check_gate(rep, paradigm, P, s, r)
    # one clock for the whole cluster: the decisions are taken in ticket
    # order, so their timestamps -- read on whichever GPU ran the push,
    # shifted onto the server GPU's clock -- never go back by more than the
    # calibration error, and all of them lie inside the run
    now = rep.decisions["now"]
    assert np.all(np.diff(now) > -50e-6), np.diff(now).min()
    assert 0 <= now.min() and now.max() <= rep.wall_s + 0.05, (now.min(), now.max(), rep.wall_s)
    w, snaps = _replay(rep, rings, d, oracle.initial_weights_f64(0, d).astype(np.float32), 0.05)
    assert np.array_equal(eng.read()[0].view(np.uint32), w.view(np.uint32))
    for p in range(P):
        last = rep.pulls[rep.pulls["worker"] == p][-1]
        mine = workers[p].params[:d].cpu().numpy()
        assert np.array_equal(mine.view(np.uint32), snaps[int(last["version"])].view(np.uint32)), p
    if paradigm in ("bsp", "ssp"):
        assert rep.defers() > 0
    eng.close()


def test_dssp_waits_less_than_ssp_on_device_flags():
    """The paper's claim on a throttled cluster (tests/test_acceptance.py:137-160
    in spirit): the fast worker waits less under DSSP(3,12) than SSP(3)."""
    waits = {}
    for paradigm, s, r in (("dssp", 3, 12), ("ssp", 3, 0)):
        eng, cl, _, _ = _synthetic_cluster(paradigm, s, r, 3, 4099, 2, [0, 50, 150])
        rep = cl.run(60)
        _check_gate(rep, paradigm, 3, s, r)
        waits[paradigm] = rep.wait_s(0)
        eng.close()
    assert waits["dssp"] < waits["ssp"], waits


def test_rejected_update_and_divergence_on_device_flags():
    P, d, K = 2, 1027, 2
    rings = []
    for p in range(P):
        ring = np.zeros((K, 1028), dtype=np.float32)
        for k in range(K):
            ring[k, :d] = oracle.synthetic_update(2, p, k, d)
        rings.append(ring)
    rings[1][1, 5] = np.nan  # worker 1's odd pushes are rejected (server.py:65-67)
    workers = [SyntheticWorker(torch.from_numpy(r).cuda()) for r in rings]
    eng = Engine("asp", P, 0, 0, 0.05, d, w0=oracle.initial_weights_f64(0, d))
    cl = FreeRunningCluster(eng, workers, graphs=True)
    cl.capture(warmup=0)
    for wk in workers:
        wk.idx.zero_()
    rep = cl.run(10)
    assert int(np.sum(rep.decisions["applied"] == 0)) == 5
    eng.refresh()
    assert eng.state.rejected == 5
    w, _ = _replay(rep, rings, d, oracle.initial_weights_f64(0, d).astype(np.float32), 0.05)
    assert np.array_equal(eng.read()[0].view(np.uint32), w.view(np.uint32))
    eng.close()
    # a finite update whose result overflows: DivergenceError, every stream
    # released (no hang), weights unchanged at the failing push
    w0 = oracle.initial_weights_f64(0, d)
    w0[3] = 3.0e38
    ring = np.zeros((1, 1028), dtype=np.float32)
    ring[0, 3] = -3.4e38
    workers = [SyntheticWorker(torch.from_numpy(ring).cuda()) for _ in range(P)]
    eng = Engine("bsp", P, 0, 0, 0.5, d, w0=w0)
    cl = FreeRunningCluster(eng, workers, graphs=True)
    cl.capture(warmup=0)
    with pytest.raises(ps.DivergenceError):
        cl.run(5)
    got, version = eng.read()
    assert version == 0
    assert np.array_equal(got.view(np.uint32), w0.astype(np.float32).view(np.uint32))
    eng.close()


def test_abort_releases_a_parked_worker():
    """BSP with one worker running alone: its first push is deferred and its
    stream parks on the go flag; ps_workers_abort (ThreadedRun.abort,
    runner.py:110-111) raises every flag and the stream drains."""
    d = 64
    ring = torch.zeros(1, 64, device="cuda")
    workers = [SyntheticWorker(ring) for _ in range(2)]
    eng = Engine("bsp", 2, 0, 0, 0.05, d)
    cl = FreeRunningCluster(eng, workers, graphs=False)
    cl._check(cl.lib.ps_workers_start(eng.handle, 1024, 1.0))
    with torch.cuda.stream(cl.streams[0]):
        cl._iteration(0, cl.streams[0].cuda_stream)
    import time
    time.sleep(0.2)
    assert not cl.streams[0].query()  # parked on the device flag
    cl.abort()
    cl.streams[0].synchronize()
    rep = cl.report()
    assert rep.aborted and rep.decision_sequence()[0][2] == "defer"
    eng.close()


def test_torch_resnet_workers_on_device_flags():
    """Four real CIFAR ResNet-20 workers on one GPU, throttled 1x/1x/2x/4x by a
    device busy-wait, DSSP(3,12): decisions equal the oracle gate's on the
    recorded sequence, the weights equal the fp32 replay of the recorded
    gradients in ticket order, and there is no host sync per iteration."""
    from paper_1908_11848_b200.workers import CifarResNet, TorchWorker, synthetic_cifar
    torch.manual_seed(0)
    P, iters = 4, 12
    workers = [TorchWorker(p, CifarResNet(20), synthetic_cifar(1, 64, seed=p)) for p in range(P)]
    d = workers[0].dimension
    w0 = workers[0].params[:d].detach().cpu().numpy().astype(np.float64)
    for wk in workers[1:]:
        wk.params.copy_(workers[0].params)
    eng = Engine("dssp", P, 3, 12, 0.01, d, w0=w0)
    rings = [torch.zeros(iters, workers[0].params.numel(), device="cuda") for _ in range(P)]
    base_us = 2000
    cl = FreeRunningCluster(eng, workers, throttle_ns=[0, 0, base_us * 1000, 3 * base_us * 1000])
    for p in range(P):
        cl.record(p, rings[p])
    cl.capture(warmup=2)
    rep = cl.run(iters)
    assert rep.pushes == P * iters
    _check_gate(rep, "dssp", P, 3, 12)
    w, _ = _replay(rep, [r.cpu().numpy() for r in rings], d, w0.astype(np.float32), 0.01)
    assert np.array_equal(eng.read()[0].view(np.uint32), w.view(np.uint32))
    assert np.all(np.isfinite(w))
    eng.close()


def test_torch_resnet_workers_on_peer_gpus():
    """Real ResNet-20 workers on different GPUs of the box (server on GPU 0),
    throttled 1x/2x/4x: the recorded gradients replayed in ticket order give
    the server's weights bit for bit; decisions equal the oracle gate's."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_1908_11848_b200.workers import CifarResNet, TorchWorker, synthetic_cifar
    torch.manual_seed(0)
    P, iters = 3, 8
    devs = [p % n for p in range(P)]
    workers = [TorchWorker(p, CifarResNet(20), synthetic_cifar(1, 32, seed=p, device=f"cuda:{devs[p]}"),
                           device=f"cuda:{devs[p]}") for p in range(P)]
    d = workers[0].dimension
    w0 = workers[0].params[:d].detach().cpu().numpy().astype(np.float64)
    for wk in workers[1:]:
        wk.params.copy_(workers[0].params.to(wk.params.device))
    eng = Engine("dssp", P, 3, 12, 0.01, d, w0=w0, device=0)
    rings = [torch.zeros(iters, workers[p].params.numel(), device=f"cuda:{devs[p]}") for p in range(P)]
    cl = FreeRunningCluster(eng, workers, throttle_ns=[0, 1_000_000, 3_000_000])
    for p in range(P):
        cl.record(p, rings[p])
    cl.capture(warmup=1)
    rep = cl.run(iters)
    assert rep.pushes == P * iters
    _check_gate(rep, "dssp", P, 3, 12)
    w, _ = _replay(rep, [r.cpu().numpy() for r in rings], d, w0.astype(np.float32), 0.01)
    assert np.array_equal(eng.read()[0].view(np.uint32), w.view(np.uint32))
    eng.close()


def test_deadline_aborts_a_run_that_cannot_finish():
    """BSP where worker 1 never gets iterations enqueued: worker 0 parks on
    its go flag forever. The host wait polls the streams and, past the
    deadline, aborts like deadline_guard (runner.py:294-298): the run ends,
    reports worker 0 as stuck, and the host never hangs."""
    d = 64
    ring = torch.zeros(1, 64, device="cuda")
    workers = [SyntheticWorker(ring) for _ in range(2)]
    eng = Engine("bsp", 2, 0, 0, 0.05, d)
    cl = FreeRunningCluster(eng, workers, graphs=False)
    cl._check(cl.lib.ps_workers_start(eng.handle, 1024, 1.0))
    import time
    t0 = time.perf_counter()
    with torch.cuda.stream(cl.streams[0]):
        for _ in range(3):
            cl._iteration(0, cl.streams[0].cuda_stream)
    stuck = cl._wait(t0, deadline_s=0.5)
    assert stuck == [0]
    rep = cl.report()
    assert rep.aborted and rep.defers(0) >= 1
    eng.close()
