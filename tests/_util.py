"""Shared test helpers (test infrastructure)."""
import synth
from oracle import chain as OC


def margin_inputs(n, B, d, dtype, seed=0, margin=1e-5, tries=64):
    """Seeded chain inputs whose ReLU inputs all stay > `margin` (relative) away from the
    decision point 0 (reading A20), so fp32 device and fp64 oracle take the same mask."""
    for s in range(seed, seed + tries):
        inp = synth.chain_inputs(n, B, d, dtype=dtype, seed=s)
        P = OC.Params(inp["W"], inp["b"], inp["gamma"], inp["beta"])
        if OC.relu_margin(P, inp["x0"], "bf16" if dtype == "bf16" else "f64") > margin:
            return inp
    raise RuntimeError("no seed with enough ReLU margin")


def assert_close(got, ref, tol, name=""):
    """Element-wise parity (reading A12): every element satisfies
    |got - ref| <= tol * (|ref| + rms(ref)), and the per-tensor relative L2 error is <= tol.
    Returns (max_abs_err, rms_ref, rel_l2) so callers can report them."""
    import numpy as np
    g = np.asarray(got, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    assert g.shape == r.shape, (name, g.shape, r.shape)
    rms = float(np.sqrt(np.mean(r * r))) if r.size else 0.0
    err = np.abs(g - r)
    bound = tol * (np.abs(r) + rms)
    bad = err > bound
    rel = float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30))
    if bad.any():
        i = np.unravel_index(int(np.argmax(err - bound)), err.shape)
        raise AssertionError(f"{name}: {int(bad.sum())} of {bad.size} elements outside tol {tol}: worst at {i} "
                             f"got {g[i]!r} ref {r[i]!r} (max_abs {err.max():.3e}, rms_ref {rms:.3e}, rel_l2 {rel:.3e})")
    assert rel <= tol, (name, rel)
    return float(err.max()) if err.size else 0.0, rms, rel
