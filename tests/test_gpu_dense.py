"""Dense building blocks of the step (csrc/dense.cu) against numpy: the
tall-skinny products X K (rowmix, DMMA and scalar paths) and the mass Gram
sum_c coeff_c A_c^T M B_c (mgram, DMMA path) over shapes that exercise the
tile padding, strided operands and multi-tile outputs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_18705_b200.build import build

    build()


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("n,kx,ky,ldx,beta", [
    (1000, 16, 16, 16, 0.0), (1000, 16, 1, 16, 0.0), (997, 13, 11, 13, 0.0),
    (50, 5, 3, 5, 0.0), (5000, 32, 16, 32, 0.0), (333, 40, 20, 40, 0.0),
    (4096, 8, 8, 24, 0.5), (1003, 16, 16, 16, -1.25), (70, 3, 9, 7, 0.0),
    # wide operands (rowmix_wide_kernel): r = 32 .. 128, ragged and strided
    (100000, 64, 64, 64, 0.0), (4099, 64, 1, 64, 0.0), (3001, 128, 128, 128, 0.5),
    (2000, 96, 70, 100, -1.0), (1000, 32, 32, 32, 0.0), (777, 12, 40, 12, 0.0),
    (5003, 64, 33, 66, 0.0), (640, 17, 24, 17, 0.0)])
def test_rowmix_matches_numpy(n, kx, ky, ldx, beta):
    from paper_2601_18705_b200.lowrank import rowmix

    rng = np.random.default_rng(n + kx + ky)
    Xf = rng.standard_normal((n, ldx))
    K = rng.standard_normal((kx, ky))
    Y0 = rng.standard_normal((n, ky))
    Xd = torch.as_tensor(Xf, device="cuda")[:, :kx]
    out = torch.as_tensor(Y0, device="cuda").clone()
    rowmix(Xd, K, out=out, beta=beta)
    ref = Xf[:, :kx] @ K + beta * Y0
    assert _rel(out.cpu().numpy(), ref) <= 1e-14


@pytest.mark.parametrize("nx,ny,ra,rb,same,with_coeff", [
    (12, 9, 16, 16, True, False), (12, 9, 16, 16, False, True), (7, 5, 5, 19, False, False),
    (20, 17, 20, 20, True, True), (33, 4, 1, 1, True, False), (9, 9, 8, 3, False, True),
    # wide bases (mgram_wide_kernel, 32- and 64-wide output blocks)
    (40, 30, 64, 64, True, False), (33, 20, 64, 64, False, True), (25, 25, 40, 40, True, True),
    (20, 20, 128, 128, True, False), (17, 9, 64, 37, False, False), (31, 31, 100, 20, False, True),
    (128, 96, 64, 64, True, True)])
def test_mass_gram_matches_numpy(nx, ny, ra, rb, same, with_coeff):
    from paper_2601_18705_b200.lowrank import mass_gram
    from paper_2601_18705_b200.mesh import build_grid, cell_blocks

    g = build_grid(nx, ny)
    M = np.asarray(cell_blocks(g)["mass"], dtype=float).reshape(4, 4)
    rng = np.random.default_rng(nx * ny + ra)
    A = rng.standard_normal((g.n_dofs, ra))
    B = A if same else rng.standard_normal((g.n_dofs, rb))
    coeff = rng.uniform(0.5, 2.0, g.n_cells) if with_coeff else None
    Ad = torch.as_tensor(A, device="cuda")
    Bd = Ad if same else torch.as_tensor(B, device="cuda")
    G = mass_gram(g, Ad, None if same else Bd, coeff).cpu().numpy()
    Ac = A.reshape(g.n_cells, 4, ra)
    Bc = B.reshape(g.n_cells, 4, -1)
    w = np.ones(g.n_cells) if coeff is None else coeff
    ref = np.einsum("c,cai,ab,cbj->ij", w, Ac, M, Bc)
    assert _rel(G, ref) <= 1e-13


@pytest.mark.parametrize("n,r,inplace", [(1000, 17, False), (4099, 32, True), (5003, 33, False),
                                        (100000, 64, True), (3001, 100, False), (2048, 128, True),
                                        (777, 128, False), (70, 48, True)])
def test_rowmix_upper_matches_numpy(n, r, inplace):
    """The triangular product of the CholQR2 step (the zero blocks of R^-1
    skipped), in place as the lean engine runs it and out of place."""
    from paper_2601_18705_b200.lowrank import rowmix_upper

    rng = np.random.default_rng(n + r)
    X = rng.standard_normal((n, r))
    K = np.triu(rng.standard_normal((r, r)))
    Xd = torch.as_tensor(X, device="cuda").clone()
    out = rowmix_upper(Xd, K, out=Xd if inplace else None)
    if inplace:
        assert out.data_ptr() == Xd.data_ptr()
    assert _rel(out.cpu().numpy(), X @ K) <= 1e-14
