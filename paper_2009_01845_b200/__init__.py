"""qsb200: a B200-native (sm_100a) dense state-vector simulator behind the qsim API.

Drop-in for the hot path of the reference simulator (arXiv 2009.01845 / Qibo re-implementation
`qsim`, /root/reference/pkg/src/qsim): states live in HBM, gates run as hand-written CUDA
kernels (single-gate kernels and fused multi-gate register-tile passes), measurement sampling
is bit-compatible with numpy's, and states larger than one GPU are sharded over ranks by global
qubits with NCCL exchanges.  Host-side objects (GateSpec, Circuit, TrotterHamiltonian, ...)
mirror the reference names and error behaviour.
"""

from .circuit import (
    CircuitGraph,
    Circuit,
    FusedGate,
    circuit_from_dict,
    circuit_to_dict,
    fuse,
    qft_circuit,
    random_grid_circuit,
    variational_circuit,
)
from .errors import ArityError, CapacityError, FormError, ParseError, ShapeError, SimulationError
from .evolution import (
    adiabatic_evolve_sharded,
    evolve_sharded,
    Callback,
    EnergyCallback,
    EntanglementEntropyCallback,
    EvolutionConfig,
    OverlapCallback,
    Schedule,
    ScheduleForm,
    Solver,
    adiabatic_evolve,
    entanglement_entropy,
    evolve,
    trotter_step_circuit,
)
from .gates import (
    CNOT,
    CZ,
    RX,
    RY,
    RZ,
    SWAP,
    CZPow,
    GateKind,
    GateSpec,
    H,
    KernelClass,
    Unitary,
    VariationalLayer,
    X,
    Y,
    Z,
    apply_gate,
    apply_matrix,
    classify_kernel,
    expanded_matrix,
    gate_matrix,
)
from .hamiltonians import (
    Form,
    TrotterHamiltonian,
    build_tfim,
    build_x,
    combine,
    expectation,
    ground_state_vector,
)
from .measurement import MeasurementResult, collapse, frequencies, marginal_probabilities, measure, sample
from .state import (
    MAX_QUBITS,
    Precision,
    StateVector,
    basis_state,
    from_amplitudes,
    max_qubits,
    norm,
    overlap,
    set_max_qubits,
    uniform_state,
    zero_state,
)

__version__ = "0.1.0"


def __getattr__(name):
    # the sharded executor pulls in torch.distributed; import it lazily
    if name in ("ExecutionPlan", "ShardedState", "execute_sharded", "gather", "partition", "plan", "reshuffle",
                "Reshuffle", "LocalSegment", "execute_distributed", "Exchange", "plan_batched"):
        from . import sharding

        return getattr(sharding, name)
    raise AttributeError(name)
