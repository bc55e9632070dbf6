"""Shared comparison of one GPU sweep with the oracle's sweep of the same input (P1).

The north_star bar is a relative Frobenius difference <= 1e-10 over the whole n x k block.  Because
the top k rows (written by kxk_finish) and the rows > k (pass C) come from different kernels, a
localised error in one block could hide under sqrt(k) ||X||_F at large k, so each block is also
checked per column: max |X_gpu - X_oracle| <= max(1e-10, u ||A||_inf / min gap).  The second term is
the first-order sensitivity of the top block: E_ij = V_ij / (d_j - d_i) (eq. Eoffdiag) turns the O(u ||A||)
rounding of V (any summation order) into u ||A|| / gap per entry -- e.g. 1.6e-9 for
k = 128 targets 5e-5 apart; the whole-block Frobenius bar stays 1e-10.  The statistics of the sweep
 are compared too, including min_gap."""
import numpy as np

TOL = 1e-10
U = 2.0 ** -53


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def cond_tol(ref, normA, tol=TOL, delta_c=10.0):
    """max(tol, u ||A||_inf / min |d_i - d_j|) over the pairs that take the 1/gap formula (gap > delta;
    pairs within delta take beta and are not amplified), from the oracle's Rayleigh quotients."""
    d = ref.debug.get("dtilde") if ref.debug else None
    if d is None or normA is None or len(d) < 2:
        return tol
    g = np.abs(d[:, None] - d[None, :])
    g = g[g > delta_c * normA * U]
    if g.size == 0:
        return tol
    return max(tol, U * normA / float(g.min()))


def compare_sweep(Xg, ref, st=None, k=None, top=True, stats_tol=1e-8, corr_rel=1e-6, corr_abs=1e-9, tol=TOL,
                  where="", normA=None, elem_tol=None):
    """Xg: the GPU's output (numpy n_loc x k); ref: oracle.SweepResult of the same input; st: the GPU's
    refine_sweep_stats (or None); top: Xg's first k rows are the global top block.  Returns the
    relative Frobenius difference."""
    k = Xg.shape[1] if k is None else k
    e = rel(Xg, ref.X)
    assert e <= tol, f"{where} one-step rel diff {e:.3e}"
    D = np.abs(Xg - ref.X)
    cn = np.maximum(np.linalg.norm(ref.X, axis=0), 1e-300)
    blocks = [(slice(0, k), "top"), (slice(k, None), "lower")] if top else [(slice(0, None), "all")]
    et = elem_tol if elem_tol is not None else cond_tol(ref, normA, tol)
    for sl, name in blocks:
        if D[sl].size:
            m = float((D[sl].max(axis=0) / cn).max())
            assert m <= et, f"{where} {name} block max-abs per column {m:.3e} (bound {et:.3e})"
    if st is not None:
        rs = ref.stats
        assert st.flipped == rs.flipped, where
        assert st.delta_hits == rs.delta_hits, (where, st.delta_hits, rs.delta_hits)
        assert abs(st.rel_resid - rs.rel_resid) <= stats_tol * max(rs.rel_resid, 1e-300) + 1e-18, where
        # ||E_L||_F carries the same 1/gap-amplified rounding as X~ (absolute floor 1e-9 ~ 1e-10 ||X||_F)
        assert abs(st.corr_norm - rs.corr_norm) <= corr_rel * rs.corr_norm + corr_abs, \
            (where, st.corr_norm, rs.corr_norm, corr_rel)
        if "dtilde" in ref.debug:
            dmax = float(np.abs(ref.debug["dtilde"]).max())
        else:
            dmax = max(abs(rs.min_gap), 1.0) * 1e3
        assert abs(st.min_gap - rs.min_gap) <= 1e-13 * dmax + 1e-300, (where, st.min_gap, rs.min_gap)
    return e
