"""One host thread per GPU (the multi-GPU control plane of SURVEY §8(e)):
the library keeps no process-wide device state, so plans built and run concurrently from
several threads -- on one device here, on devices 0 and 1 when two GPUs are visible -- give
the same bytes as a single-threaded run."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200.abi import PB_BF16  # noqa: E402
from paper_2312_05516_b200.workloads import SplitMix64, _build  # noqa: E402


def _work(seed):
    rng = SplitMix64(seed)
    convs = [[(0, 200)], [(700, 1)], [(64, 130)], [(1500, 1)], [(3000, 1)]]
    return _build("thr", 32, 4, 128, 16, PB_BF16, rng.seed, convs, rng)


def _run_on(gh, torch, dev, w, results, key, barrier):
    torch.cuda.set_device(dev)
    q, k, v = gh.device_inputs(w, dev=f"cuda:{dev}")
    barrier.wait()
    outs = []
    for _ in range(3):
        got, _ = gh.run_plan(w, q, k, v)
        outs.append(got)
    results[key] = outs


def _threads(gh, torch, devices):
    w = [_work(11 + i) for i in range(len(devices))]
    results = {}
    barrier = threading.Barrier(len(devices))
    ts = [threading.Thread(target=_run_on, args=(gh, torch, d, w[i], results, i, barrier)) for i, d in
          enumerate(devices)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    # single-threaded references
    for i, d in enumerate(devices):
        torch.cuda.set_device(d)
        q, k, v = gh.device_inputs(w[i], dev=f"cuda:{d}")
        ref, _ = gh.run_plan(w[i], q, k, v)
        for got in results[i]:
            assert np.array_equal(got, ref)
    torch.cuda.set_device(0)


def test_two_threads_one_device(cuda):
    import gpu_helpers as gh
    _threads(gh, cuda, [0, 0])


def test_one_thread_per_device(cuda):
    if cuda.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import gpu_helpers as gh
    _threads(gh, cuda, [0, 1])
