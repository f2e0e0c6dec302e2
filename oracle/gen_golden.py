"""Generate tests/golden/*.npz from the REAL reference simulator (test infrastructure only).

Run in the build container, where /root/reference is mounted read-only:
    python oracle/gen_golden.py
The fixtures pin both the CPU oracle (oracle/statevec.py) and the CUDA path; the GPU box never
needs /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import oracle as ref_oracle  # noqa: E402  (reference's own test oracle: random gates/states)
import qsim  # noqa: E402
from qsim.circuit import circuit_to_dict  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
import importlib.util  # noqa: E402

_spec = importlib.util.spec_from_file_location("qsb_oracle_statevec", os.path.join(HERE, "statevec.py"))
ov = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(ov)


def to_ref_circuit(n, gates):
    c = qsim.Circuit(n)
    for kind, tg, ct, params, m in gates:
        if kind == "Unitary":
            c.add(qsim.Unitary(m, *tg, controls=ct))
        else:
            c.add(qsim.GateSpec(qsim.GateKind(kind), tg, ct, params))
    return c


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)


def circ_json(c):
    return np.array(json.dumps(circuit_to_dict(c)))


def main():
    rng = np.random.default_rng(2009_01845)

    # 1. single random gates (all kinds, up to 3 controls) at n = 8, reference test oracle generator
    singles = []
    for i in range(60):
        spec = ref_oracle.random_gate(8, rng, max_controls=3)
        init = ref_oracle.random_state(8, rng)
        c = qsim.Circuit(8).add(spec)
        out = c.execute(init)
        singles.append((json.dumps(circuit_to_dict(c)), init.amplitudes, out.amplitudes))
    save("single_gates", circuits=np.array([s[0] for s in singles]), inputs=np.stack([s[1] for s in singles]),
         outputs=np.stack([s[2] for s in singles]))

    # 2. random circuits (depth 40, <= 2 controls), n in {10, 13, 14}
    rc = []
    for n in (10, 13, 14):
        for k in range(3):
            c = ref_oracle.random_circuit(n, 40, rng, max_controls=2)
            init = ref_oracle.random_state(n, rng)
            rc.append((n, json.dumps(circuit_to_dict(c)), init.amplitudes, c.execute(init).amplitudes))
    save("random_circuits", n=np.array([r[0] for r in rc]), circuits=np.array([r[1] for r in rc]),
         **{f"in{i}": r[2] for i, r in enumerate(rc)}, **{f"out{i}": r[3] for i, r in enumerate(rc)})

    # 3. QFT
    q = {}
    for n in (10, 14):
        c = qsim.qft_circuit(n)
        q[f"zero{n}"] = c.execute().amplitudes
        k = int(np.random.default_rng(42).integers(1 << n))
        basis = np.zeros(1 << n, dtype=complex)
        basis[k] = 1.0
        q[f"basisk{n}"] = np.array(k)
        q[f"basis{n}"] = c.execute(qsim.from_amplitudes(basis)).amplitudes
        init = ref_oracle.random_state(n, np.random.default_rng(42))
        q[f"rin{n}"] = init.amplitudes
        q[f"rout{n}"] = c.execute(init).amplitudes
        q[f"f32_{n}"] = c.execute(precision=qsim.Precision.F32).amplitudes
    save("qft", **q)

    # 4. variational (cli.py:179-181 parameters), fused and unfused, c128 and c64
    v = {}
    for n in (10, 14):
        params = np.random.default_rng(42).uniform(0, 2 * np.pi, n * (2 * 3 + 1))
        v[f"params{n}"] = params
        for fused in (False, True):
            c = qsim.variational_circuit(n, 3, params, fused=fused)
            v[f"f64_{n}_{int(fused)}"] = c.execute().amplitudes
            v[f"f32_{n}_{int(fused)}"] = c.execute(precision=qsim.Precision.F32).amplitudes
    save("variational", **v)

    # 5. supremacy-style grid circuit (3 x 5 = 15 qubits, 8 cycles), defined in oracle/statevec.py
    gates = ov.grid_supremacy(3, 5, 8, seed=42)
    c = to_ref_circuit(15, gates)
    save("grid15", circuit=circ_json(c), out=c.execute().amplitudes)

    # 6. Trotter adiabatic evolution (build_x -> build_tfim(h=1), linear schedule)
    from qsim.evolution import EvolutionConfig, Schedule, Solver, adiabatic_evolve
    from qsim.hamiltonians import Form, build_tfim, build_x

    adi = {}
    for n, dt, T in ((8, 0.05, 0.5), (13, 0.1, 0.5), (14, 0.1, 0.3)):
        h0 = build_x(n, Form.TROTTER)
        h1 = build_tfim(n, 1.0, Form.TROTTER)
        st = adiabatic_evolve(h0, h1, Schedule.linear(), EvolutionConfig(Solver.TROTTER, dt, T))
        adi[f"n{n}"] = st.amplitudes
        adi[f"cfg{n}"] = np.array([dt, T])
    save("adiabatic", **adi)

    # 7. sampling: marginals (bitwise) and samples for several qubit subsets and seeds
    smp = {}
    n = 12
    init = ref_oracle.random_state(n, np.random.default_rng(7))
    smp["state"] = init.amplitudes
    subsets = [tuple(range(n)), (0,), (11,), (0, 1, 2), (3, 7), (11, 0, 5), (2, 4, 6, 8, 10), tuple(range(1, 12)),
               (5, 6, 7, 8), tuple(reversed(range(n)))]
    smp["subsets"] = np.array([json.dumps(s) for s in subsets])
    for i, s in enumerate(subsets):
        smp[f"marg{i}"] = qsim.marginal_probabilities(init, s)
        smp[f"samp{i}"] = qsim.sample(init, s, 2000, seed=100 + i).samples
    f32 = qsim.StateVector(n, init.amplitudes.astype(np.complex64), qsim.Precision.F32)
    smp["marg_f32"] = qsim.marginal_probabilities(f32, (0, 3, 5))
    smp["samp_f32"] = qsim.sample(f32, (0, 3, 5), 1000, seed=9).samples
    # CLI shots digests (cli.py:193-212): H on every qubit, then sample all qubits
    for nq, shots, seed in ((3, 500, 7), (20, 100000, 42)):
        c = qsim.Circuit(nq).add([qsim.H(k) for k in range(nq)])
        res = qsim.sample(c.execute(), range(nq), shots, seed)
        smp[f"digest_{nq}_{shots}_{seed}"] = np.array(hashlib.sha256(res.samples.tobytes()).hexdigest())
    save("sampling", **smp)

    # 8. sharded execution (reference execute_sharded == execute) on QFT-14 and a random circuit
    from qsim.sharding import execute_sharded, plan

    sh = {}
    c = qsim.qft_circuit(14)
    for shards in (2, 4, 8):
        p = plan(c, shards)
        sh[f"qft14_reshuffles_{shards}"] = np.array(p.n_reshuffles)
        sh[f"qft14_globals_{shards}"] = np.array(p.global_qubits)
    save("sharding", **sh)
    print("golden fixtures written to", OUT)


def main_c64_large():
    """complex64 fixtures at n = 16 (512 KB states): above the 128 KB shared-memory batch limit,
    so the planned fused passes (packed FP32-pair code) run against the reference itself."""
    rng = np.random.default_rng(16_64)
    out = {}
    n = 16
    c = qsim.qft_circuit(n)
    init = ref_oracle.random_state(n, rng)
    f32 = qsim.StateVector(n, init.amplitudes.astype(np.complex64), qsim.Precision.F32)
    out["qft_in"] = f32.amplitudes
    out["qft_out"] = c.execute(f32, precision=qsim.Precision.F32).amplitudes
    params = np.random.default_rng(42).uniform(0, 2 * np.pi, n * (2 * 3 + 1))
    out["var_params"] = params
    for fused in (False, True):
        vc = qsim.variational_circuit(n, 3, params, fused=fused)
        out[f"var_{int(fused)}"] = vc.execute(precision=qsim.Precision.F32).amplitudes
    gates = ov.grid_supremacy(4, 4, 8, seed=7)
    gc = to_ref_circuit(n, gates)
    out["grid_circuit"] = circ_json(gc)
    out["grid_out"] = gc.execute(precision=qsim.Precision.F32).amplitudes
    save("c64_large", **out)
    print("c64_large fixture written to", OUT)


if __name__ == "__main__":
    if sys.argv[1:] == ["c64_large"]:
        main_c64_large()
    else:
        main()
        main_c64_large()
