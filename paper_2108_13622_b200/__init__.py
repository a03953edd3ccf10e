"""B200-native (sm_100a) Leja / FD-JVP / MHD-RHS hot path of arxiv/paper_2108_13622.

A drop-in for the reference package ``xmhd``'s hot path: the public names of
``pkg/src/xmhd/__init__.py:21-29`` that belong to the path are re-exported with
the same signatures; their work runs in hand-written fp64 CUDA kernels behind
the C-ABI ``include/xmhd_b200.h`` (``_xmhd_b200.so``).  There is no CPU
fallback: without the library or a CUDA device every compute entry point
raises ``NativeUnavailable``.
"""

from paper_2108_13622_b200._lib import NativeUnavailable
from paper_2108_13622_b200.controllers import (ControllerConstants, ControllerMode, accept,
                                               combine, cost_next, traditional_next)
from paper_2108_13622_b200.harness import (RunConfig, RunReport, StepRecord, divb_series,
                                           make_reference, run, work_precision)
from paper_2108_13622_b200.integrators import Scheme, error_norm, step
from paper_2108_13622_b200.krylov import apply_phi_krylov
from paper_2108_13622_b200.leja import (JacobianAction, PhiApplyResult, ShiftScale,
                                        apply_phi_leja, leja_points, shift_and_scale)
from paper_2108_13622_b200.linearize import (FrozenLinearization, RhsBlowupError, RhsOperator,
                                             SpectralEstimate, estimate_alpha, jvp, remainder)
from paper_2108_13622_b200.mhd import (Boundary, MHDParams, MhdRhs, StateGrid, apply_bc,
                                       conserved_totals, discrete_div_b, mhd_rhs,
                                       read_checkpoint, write_checkpoint)
from paper_2108_13622_b200.phi import divided_differences, phi_scalar

__version__ = "0.1.0"
