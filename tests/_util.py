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
