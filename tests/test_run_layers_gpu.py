"""pb_attn_run_layers: the layer loop as one CUDA graph launch.  Its outputs must be the bytes
of the same per-layer pb_attn_run launches (fused and separate-decode schedules), the graph
must read the pools at replay time, re-capture when a pointer changes, count its kernels per
launch, and nest inside a caller's own capture."""
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16, PB_F32, AttentionPlan  # noqa: E402
from paper_2312_05516_b200.workloads import SplitMix64, random_instance  # noqa: E402

L = 4


@pytest.fixture(scope="module")
def gh(cuda):
    import gpu_helpers as gh
    return gh


def _layers(gh, w):
    ks, vs = [], []
    for l in range(L):
        q, k, v = gh.device_inputs(w, layer=l)
        ks.append(k)
        vs.append(v)
    return q, ks, vs


def _eager(torch, plan, q, ks, vs, ws, st):
    outs = []
    for l in range(L):
        o = torch.zeros_like(q)
        plan.run(q.data_ptr(), ks[l].data_ptr(), vs[l].data_ptr(), o.data_ptr(), ws.data_ptr(), st)
        outs.append(o)
    torch.cuda.synchronize()
    return outs


def _same(torch, a, b):
    return all(torch.equal(x.view(torch.int16), y.view(torch.int16)) for x, y in zip(a, b))


@pytest.mark.parametrize("flags,d,dtype", [(0, 128, PB_BF16), (abi.PB_PLAN_SEPARATE_DECODE, 128, PB_BF16),
                                           (0, 64, PB_BF16), (0, 128, PB_F32)])
def test_graph_layers_equal_eager_layers(gh, cuda, flags, d, dtype):
    """bf16 d = 128 (fused and separate schedules), d = 64, and the fp32 validation mode (SIMT
    kernels) inside the graph."""
    torch = cuda
    w = random_instance(SplitMix64(77), 32, 4, d, 16, dtype, 10, 2500, max_q=300)
    q, ks, vs = _layers(gh, w)
    st = torch.cuda.current_stream().cuda_stream
    plan = AttentionPlan(w.shape(), w.batch(), flags)
    plan.upload(st)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    want = _eager(torch, plan, q, ks, vs, ws, st)
    outs = [torch.zeros_like(q) for _ in range(L)]
    args = ([q.data_ptr()] * L, [k.data_ptr() for k in ks], [v.data_ptr() for v in vs],
            [o.data_ptr() for o in outs])
    n0 = abi.launch_count()
    plan.run_layers(*args, ws.data_ptr(), st)   # captures, then launches
    torch.cuda.synchronize()
    assert _same(torch, outs, want)
    per_call = abi.launch_count() - n0
    assert per_call >= L  # one kernel per layer at least, counted once per launch
    for o in outs:
        o.zero_()
    plan.run_layers(*args, ws.data_ptr(), st)   # replay
    torch.cuda.synchronize()
    assert _same(torch, outs, want)
    assert abi.launch_count() - n0 == 2 * per_call

    # the graph reads the pools when it runs: new contents, same pointers
    abi.fill_unit(ks[1].data_ptr(), dtype, w.pool_elems, w.seed + 1, 0)
    want2 = _eager(torch, plan, q, ks, vs, ws, st)
    plan.run_layers(*args, ws.data_ptr(), st)
    torch.cuda.synchronize()
    assert _same(torch, outs, want2)
    assert not torch.equal(want2[1].view(torch.int16), want[1].view(torch.int16))

    # a pointer change re-captures: layers in reverse order
    rk, rv = ks[::-1], vs[::-1]
    want3 = _eager(torch, plan, q, rk, rv, ws, st)
    plan.run_layers([q.data_ptr()] * L, [k.data_ptr() for k in rk], [v.data_ptr() for v in rv],
                    [o.data_ptr() for o in outs], ws.data_ptr(), st)
    torch.cuda.synchronize()
    assert _same(torch, outs, want3)


def test_run_layers_inside_a_callers_capture(gh, cuda):
    torch = cuda
    w = random_instance(SplitMix64(78), 16, 2, 128, 16, PB_BF16, 8, 2000, max_q=200)
    q, ks, vs = _layers(gh, w)
    side = torch.cuda.Stream()
    plan = AttentionPlan(w.shape(), w.batch())
    plan.upload(side.cuda_stream)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    want = _eager(torch, plan, q, ks, vs, ws, torch.cuda.current_stream().cuda_stream)
    outs = [torch.zeros_like(q) for _ in range(L)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        plan.run_layers([q.data_ptr()] * L, [k.data_ptr() for k in ks], [v.data_ptr() for v in vs],
                        [o.data_ptr() for o in outs], ws.data_ptr(), side.cuda_stream)
    for _ in range(2):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert _same(torch, outs, want)
