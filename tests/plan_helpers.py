"""Test helpers: execute a fusion Plan on CPU with the pass emulator + oracle kernels."""

import numpy as np

from oracle import statevec as ov
from pass_emulator import run_program


def spec_tuples_to_specs(gates):
    """oracle gate tuples -> package GateSpecs (for the planner)."""
    from paper_2009_01845_b200 import gates as G

    out = []
    for kind, tg, ct, params, m in gates:
        if kind == "Unitary":
            out.append(G.Unitary(m, *tg, controls=ct))
        else:
            out.append(G.GateSpec(G.GateKind(kind), tg, ct, params))
    return out


def emulate_plan(plan, psi, dtype=np.complex128):
    from paper_2009_01845_b200.fusion import GateStep, PassStep

    n = plan.n_qubits
    psi = np.array(psi, dtype=dtype, copy=True)
    for st in plan.steps:
        if isinstance(st, PassStep):
            psi = run_program(psi, st.words, dtype)
        else:
            g = st.gate
            tq = tuple(n - 1 - b for b in g.targets)
            cq = tuple(n - 1 - b for b in g.controls)
            if g.kind == "diag":
                m = np.diag(g.matrix)
            elif g.kind == "swap":
                m = ov.FIXED["SWAP"]
            else:
                m = g.matrix
            ov.apply_matrix(psi, n, tq, m, cq)
    return psi
