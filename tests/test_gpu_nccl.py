"""The NCCL gradient-allreduce path on one GPU: a single-rank
communicator attached to a solver runs the same device pipeline as the
multi-GPU case (dlopen'ed NCCL, ncclAllReduce of the gradient sum + record
count on the solver stream before Adam). With one rank the allreduce is the
identity, so training must behave exactly like the solver without a
communicator: same number of Adam steps and the same records consumed, and
parameters within fp32 atomic-order noise."""
import numpy as np
import pytest

from paper_2410_18944_b200 import abi, api
from paper_2410_18944_b200.scene import cell_centers, make_preset

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mlp", [api.MLP_TENSOR, api.MLP_EXACT])
def test_single_rank_nccl_training_matches_local(gpu, mlp):
    p = make_preset("neumann-strip-vlin")
    pts = cell_centers(64, 64, p.eval_bbox)
    out = []
    for with_comm in (False, True):
        f = api.GuidingField(abi.field_config(), p.scene.bbox, 5)
        s = api.Solver(api.Accel(p.scene), f, abi.solver_config("learnable_mis"), mlp)
        if with_comm:
            s.attach_comm(api.comm_unique_id(), 1, 0)
        s.set_points(pts)
        st, _ = s.run(1, 2, 256, abi.train_config(seed=1))
        out.append((st.steps, st.records_consumed, f.params()))
    (s0, c0, p0), (s1, c1, p1) = out
    assert s1 == s0 and c1 == c0
    assert np.all(np.isfinite(p1))
    # fp32 gradient atomics differ in order between the runs; for parameters
    # whose gradient is ~0 Adam's m / sqrt(v) can flip sign, moving them by up
    # to lr per step, so only the bulk is compared tightly
    d = np.abs(p1 - p0)
    lr = abi.train_config().lr
    assert d.max() <= 2.0 * lr * s0 + 1e-6, d.max()
    assert np.percentile(d, 99) < 1e-4 and np.median(d) < 1e-6, (np.percentile(d, 99), np.median(d))


def test_single_rank_nccl_training_matches_local_3d(gpu):
    """The 3D solver's allreduce path (wostgpu_solver3_attach_comm) with one
    rank: same Adam steps and records as without a communicator."""
    from paper_2410_18944_b200.api3 import MLP_TENSOR, Accel3, GuidingField3, Solver3
    from paper_2410_18944_b200.scene3 import make_preset3, slice_points
    p = make_preset3("box-strip-vlin", n=16)
    x = slice_points(48, 48)
    out = []
    for with_comm in (False, True):
        f = GuidingField3(abi.field_config3(), (0, 0, 0, 1, 1, 1), 5)
        s = Solver3(Accel3(p.scene), f, abi.solver_config("learnable_mis"), MLP_TENSOR)
        if with_comm:
            s.attach_comm(api.comm_unique_id(), 1, 0)
        s.set_points(x)
        st, _ = s.run(1, 2, 256, abi.train_config(seed=1))
        out.append((st.steps, st.records_consumed, f.params()))
    (s0, c0, p0), (s1, c1, p1) = out
    assert s1 == s0 and c1 == c0 and s0 >= 2
    d = np.abs(p1 - p0)
    assert np.all(np.isfinite(p1)) and d.max() <= 2.0 * abi.train_config().lr * s0 + 1e-6
