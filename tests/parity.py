"""Shared parity helpers for the GPU tests (tolerances from BASELINE.json north_star)."""
import numpy as np
import torch

FROB_TOL = 5e-3      # ||Y_gpu - Y_ref||_F / ||Y_ref||_F
ELEM_ATOL = 1e-2     # |Y_gpu - Y_ref| <= 1e-2 * (1 + |Y_ref|)


def to64(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def assert_parity(y_gpu: torch.Tensor, y_ref: np.ndarray, what: str = ""):
    g = to64(y_gpu)
    assert g.shape == y_ref.shape, (g.shape, y_ref.shape)
    assert np.all(np.isfinite(g)), f"{what}: non-finite GPU output"
    diff = g - y_ref
    nref = np.linalg.norm(y_ref)
    rel = np.linalg.norm(diff) / nref if nref > 0 else np.linalg.norm(diff)
    bound = ELEM_ATOL * (1.0 + np.abs(y_ref))
    bad = np.abs(diff) > bound
    worst = float(np.max(np.abs(diff) - bound)) if diff.size else 0.0
    assert rel <= FROB_TOL, f"{what}: relative Frobenius error {rel:.3e} > {FROB_TOL}"
    assert not bad.any(), f"{what}: {int(bad.sum())} elements exceed 1e-2(1+|ref|), worst excess {worst:.3e}"
    return rel


def sample_rows(n: int, k: int, seed: int = 1234) -> np.ndarray:
    """Seeded token-row sample (always includes the first and last row: tile edges/tails)."""
    if n <= k:
        return np.arange(n)
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(np.arange(1, n - 1), size=k - 2, replace=False))
    return np.concatenate([[0], rows, [n - 1]])
