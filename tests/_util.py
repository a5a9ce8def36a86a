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


def assert_close(got, ref, tol, name="", max_frac=0.0):
    """Element-wise parity (reading A12): every element satisfies
    |got - ref| <= tol * (|ref| + rms(ref)) — or all but a fraction max_frac of them, for deep
    recurrences where the bf16 rounding decisions of the two precisions drift apart — and the
    per-tensor relative L2 error is <= tol.  Returns (max_abs_err, rms_ref, rel_l2)."""
    import numpy as np
    g = np.asarray(got, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    assert g.shape == r.shape, (name, g.shape, r.shape)
    rms = float(np.sqrt(np.mean(r * r))) if r.size else 0.0
    err = np.abs(g - r)
    bound = tol * (np.abs(r) + rms)
    bad = err > bound
    rel = float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30))
    if bad.mean() > max_frac:
        i = np.unravel_index(int(np.argmax(err - bound)), err.shape)
        raise AssertionError(f"{name}: {int(bad.sum())} of {bad.size} elements outside tol {tol}: worst at {i} "
                             f"got {g[i]!r} ref {r[i]!r} (max_abs {err.max():.3e}, rms_ref {rms:.3e}, rel_l2 {rel:.3e})")
    assert rel <= tol, (name, rel)
    return float(err.max()) if err.size else 0.0, rms, rel


def ambiguous_features(P, x0, mode="bf16", tau=1e-3):
    """Features whose ReLU decision is ambiguous between fp32 (device) and fp64 (oracle) arithmetic
    (reading A20): per layer l, the features f with min_b |u_l[b, f]| < tau * rms(u_l), u = gamma
    xhat + beta, along the oracle's own forward pass.  A decision taken differently there moves
    dgamma_l[f], dbeta_l[f], db_{l-1}[f] and row f of dW_{l-1} (through column f of dx_l) by O(1)
    relative while every other element stays within rounding (test infrastructure)."""
    import numpy as np
    x = np.asarray(x0, dtype=np.float64)
    out = []
    for l in range(P.n):
        mu = x.mean(axis=0)
        rstd = 1.0 / np.sqrt(((x - mu) ** 2).mean(axis=0) + OC.EPS)
        u = P.gamma[l] * (x - mu) * rstd + P.beta[l]
        out.append(set(np.nonzero(np.abs(u).min(axis=0) < tau * np.sqrt(np.mean(u * u)))[0].tolist()))
        x = OC.block_forward(x, P, l, mode)
    return out


def assert_close_chain(grads, ref, P, x0, tol, tag=""):
    """Element-wise chain parity with the decision-ambiguous positions of ambiguous_features()
    excluded from the element bound (they are still inside the relative-L2 bound); returns the
    per-tensor (max_abs, rms_ref, rel_l2, n_excluded).  A decision taken differently at layer l+1
    also moves every feature of layer l's gamma / beta / db a little (through da_l = dx_{l+1} W_l):
    those per-feature vectors are held element-wise only below no ambiguous layer, else to the
    per-layer relative-L2 bound."""
    import numpy as np
    amb = ambiguous_features(P, x0)
    n = P.n
    stats = {}
    for k in ref:
        g, r = np.asarray(grads[k], np.float64), np.asarray(ref[k], np.float64)
        mask = np.ones(r.shape, dtype=bool)
        for l in range(n):
            above = any(amb[j] for j in range(l + 1, n))
            if k == "W" and l + 1 < n:
                mask[l, sorted(amb[l + 1]), :] = False
            elif k in ("gamma", "beta"):
                mask[l, sorted(amb[l])] = False
                if above:
                    mask[l, :] = False
            elif k == "b" and l + 1 < n:
                mask[l, sorted(amb[l + 1])] = False
                if any(amb[j] for j in range(l + 2, n)):
                    mask[l, :] = False
            if k != "W" and not mask[l].all():
                rl = float(np.linalg.norm(g[l] - r[l]) / max(np.linalg.norm(r[l]), 1e-30))
                assert rl <= tol, (tag, k, l, rl)
        rms = float(np.sqrt(np.mean(r * r)))
        err = np.abs(g - r)
        bad = (err > tol * (np.abs(r) + rms)) & mask
        rel = float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30))
        if bad.any():
            i = np.unravel_index(int(np.argmax(np.where(mask, err - tol * (np.abs(r) + rms), -np.inf))), err.shape)
            raise AssertionError(f"{tag} {k}: {int(bad.sum())} elements outside tol {tol} away from ambiguous ReLU "
                                 f"decisions: worst at {i} got {g[i]!r} ref {r[i]!r} (rel_l2 {rel:.3e})")
        assert rel <= tol, (tag, k, rel)
        stats[k] = (float(err[mask].max()) if mask.any() else 0.0, rms, rel, int((~mask).sum()))
    return stats
