"""Determinism and shared-workspace soak tests (GPU).

The persistent kernels take work items from global tickets, so which CTA runs an item changes
from launch to launch; each item's arithmetic does not, so repeated launches must give the same
bytes.  Self-resetting tickets and split-group counters must also survive many different plans
run one after another on one workspace buffer (the header allows sequential reuse)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2312_05516_b200 import abi  # noqa: E402
from paper_2312_05516_b200.abi import PB_BF16  # noqa: E402
from paper_2312_05516_b200.workloads import SplitMix64, config, random_instance  # noqa: E402


@pytest.fixture(scope="module")
def gh(cuda):
    import gpu_helpers as gh
    return gh


@pytest.mark.parametrize("cfg", [2, 4])
def test_repeated_launches_are_bit_identical(gh, cuda, cfg):
    torch = cuda
    w = config(cfg)
    q, k, v = gh.device_inputs(w)
    plan = abi.AttentionPlan(w.shape(), w.batch())
    st = torch.cuda.current_stream().cuda_stream
    plan.upload(st)
    ws = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(12):
        out = torch.empty_like(q)
        plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), ws.data_ptr(), st)
        outs.append(out)
    torch.cuda.synchronize()
    first = outs[0].view(torch.int16)
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16), first)


def test_many_plans_share_one_workspace(gh, cuda):
    torch = cuda
    rng = SplitMix64(424242)
    st = torch.cuda.current_stream().cuda_stream
    shared = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    layouts = [(8, 8, 128), (16, 2, 128), (64, 8, 128), (8, 1, 64), (40, 10, 128)]
    flags = [0, abi.PB_PLAN_SEPARATE_DECODE, abi.PB_PLAN_LPT_ORDER]
    for trial in range(24):
        n_head, n_kv, d = layouts[trial % len(layouts)]
        w = random_instance(rng, n_head, n_kv, d, 16, PB_BF16, 1 + rng.next() % 12, 3000,
                            all_decode=(trial % 4 == 3), max_q=400)
        q, k, v = gh.device_inputs(w)
        f = flags[trial % len(flags)]
        plan = abi.AttentionPlan(w.shape(), w.batch(), f)
        plan.upload(st)
        assert plan.workspace_bytes() <= shared.numel()
        out_shared = torch.empty_like(q)
        plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out_shared.data_ptr(), shared.data_ptr(), st)
        fresh = torch.zeros(max(1, plan.workspace_bytes()), dtype=torch.uint8, device="cuda")
        out_fresh = torch.empty_like(q)
        plan.run(q.data_ptr(), k.data_ptr(), v.data_ptr(), out_fresh.data_ptr(), fresh.data_ptr(), st)
        torch.cuda.synchronize()
        n = w.total_tokens * w.n_head * w.head_size
        assert torch.equal(out_shared[:n].view(torch.int16), out_fresh[:n].view(torch.int16)), (trial, plan.stats())
