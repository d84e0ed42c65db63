"""A numeric pass on device operands makes no host synchronisation: it is
captured into a CUDA graph and replayed (the status of each pass travels to
pinned host memory behind it, ptap_plan_status_async).  Both the default and
the deterministic pass; the replayed C equals the eager one."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("det", [False, True])
def test_numeric_pass_captures_into_cuda_graph(det):
    import torch

    import paper_1905_08423_b200 as pk
    from paper_1905_08423_b200 import devgen
    ctx = pk.single_rank_context()
    a, p = devgen.config_dist("cfg3", 1, 0, ctx.device, n_fine=32)
    plan = pk.run_symbolic(a, p, "allatonce", ctx, deterministic=det)
    _, _, v0 = pk.run_numeric_device(a, p, plan, ctx)
    want = v0.clone()
    plan.check()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        _, _, v = pk.run_numeric_device(a, p, plan, ctx)
    for _ in range(3):
        v.zero_()
        g.replay()
        torch.cuda.synchronize()
        if det:
            assert torch.equal(v.view(torch.int64), want.view(torch.int64))
        else:
            assert float((v - want).abs().max()) <= 1e-12 * float(want.abs().max())
    plan.check()
