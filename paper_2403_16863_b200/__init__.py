"""B200-native SIP: stochastic instruction perturbation for sm_100a SASS schedules.

Same public names as the reference package ``sasstune`` (reference
``__init__.py:8-118``); the search, legality, scoreboard, evaluation and
verification run on the GPU through ``libsip.so`` (include/sip.h).
"""
from .anneal import (AnnealConfig, AnnealState, HistoryRecord, InvalidBaseline, accept_move, anneal,
                     feedback)
from .backends import (BackendDescriptor, CostSample, ExternalCommandBackend, MeasurementFailed,
                       SimulatorBackend, make_backend)
from .difftest import (BufferSpec, FailureDetail, TestPlan, TestVerdict, first_failure_index, pass_curve,
                       run_tests, sample_inputs)
from .deps import DepEdge, DepGraph, DepKind, build_depgraph, mem_refs, reads_writes, swap_legal
from .driver import ChainOutcome, SearchReport, run_search
from .estimator import ScheduleTuner, as_kernel
from .ir import (ControlCode, ControlError, Instruction, InstrClass, Kernel, Operand, OperandKind,
                 classify)
from .interp import (CompiledKernel, OutOfBoundsAccess, UninitializedRead, UnsupportedInstruction,
                     interpret)
from .machine import MachineConfig, SimReport, simulate
from .perturb import (Action, CandidateSet, Direction, MoveRejected, NoCandidatesError, apply_action,
                      candidates, sample_action)
from .sasstext import ParseDiagnostic, ParseError, parse_control, parse_kernel, serialize_kernel
from .store import ResultStore, input_hash

__version__ = "0.1.0"
