"""B200-native sFISTA hot path with the kronblur solver/operator API (arXiv 1901.00913).

Drop-in entry points (same names, signatures and error behaviour as the reference package
``kronblur``): ``sfista``, ``kron_apply``, ``kron_apply_adjoint``, ``estimate_lipschitz``,
``objective_matrix``, ``decompose``, ``blur_direct``. The arithmetic of the first four runs in the sm_100a kernels of
``libkb_b200.so`` (C ABI: include/kronblur_b200.h); ``decompose`` is the one-time host setup.
``install(kronblur, options=None)`` reroutes an imported ``kronblur`` to these functions.
"""

from .blur import blur_direct, blur_direct_batch
from .errors import ArgumentError, CapacityError, FormatError, KronblurError, NumericError
from .kron import (
    KronOperator,
    KronTerm,
    decompose,
    kron_apply,
    kron_apply_adjoint,
    kron_to_dense,
    truncation_error,
)
from .psf import BoundaryCondition, Psf, pad_to, unvec, vec
from .solvers import (
    LIPSCHITZ_SAFETY,
    IterationRecord,
    SolveConfig,
    SolveOptions,
    SolveRun,
    estimate_lipschitz,
    lipschitz,
    make_ops,
    momentum_next,
    momentum_table,
    objective,
    objective_matrix,
    select_lambda,
    sfista,
    sfista_batch,
)
from .structured import FactorKind, StructuredFactor, factor_band, factor_to_dense, hank, toep, toep_plus_hank

__version__ = "0.1.0"


from .dropin import install  # noqa: E402  (patches an imported kronblur; see dropin.py)
