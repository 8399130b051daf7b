"""K9 tiled-Cholesky executor: numerics vs LAPACK fp64, schedule invariants."""
import numpy as np
import pytest
import torch

from paper_1502_07451_b200.cholesky import TiledCholesky, spd_matrix, task_table

pytestmark = pytest.mark.gpu


def test_task_table_shape():
    tb = task_table(8)
    assert tb.n_tasks == 120 and len(tb.deps) == 252
    tb = task_table(64)
    assert tb.n_tasks == 45760 and len(tb.deps) == 131040


@pytest.mark.parametrize("n", [512, 1024, 2048, 4096])
def test_factor_matches_lapack(n):
    A = spd_matrix(n, seed=1)
    L = TiledCholesky(n).factor(A)
    ref = np.linalg.cholesky(A.cpu().numpy())
    err = np.abs(L.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 1e-10, err
    # residual check on the device
    R = (L @ L.T - A).abs().max().item() / A.abs().max().item()
    assert R <= 1e-12, R


def test_repeatable():
    A = spd_matrix(2048, seed=3)
    c = TiledCholesky(2048)
    L1 = c.factor(A).clone()
    L2 = c.factor(A)
    assert torch.equal(L1, L2)


def test_not_spd_raises():
    A = -torch.eye(1024, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        TiledCholesky(1024).factor(A)


def test_config3_factor_n32768():
    """Config 3 itself (n = 32768, 64 x 64 tiles, 45,760 tasks): the leading
    4096 x 4096 block of L equals LAPACK's factor of the leading principal
    submatrix (a Cholesky factor's leading block is the factor of the leading
    block), and 64 sampled columns of L L^T reproduce A."""
    n = 32768
    A = spd_matrix(n, seed=7)
    L = TiledCholesky(n).factor(A)
    ref = np.linalg.cholesky(A[:4096, :4096].cpu().numpy())
    err = np.abs(L[:4096, :4096].cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 1e-10, err
    cols = torch.randint(0, n, (64,), generator=torch.Generator().manual_seed(1)).to(A.device)
    R = (L @ L[cols, :].T - A[:, cols]).abs().max().item() / A.abs().max().item()
    assert R <= 1e-12, R
