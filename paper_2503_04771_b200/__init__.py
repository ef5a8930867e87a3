"""paper_2503_04771_b200 — B200-native (sm_100a) backend for the einsum /
``linalg.generic`` contraction path of arXiv 2503.04771 (reference: bridgegen).

Drop-in surface (mirrors bridgegen):  ``einsum.parse_einsum``,
``einsum.derive_maps``, ``einsum.build_einsum_function``,
``interp.run_function``; ``compat.install()`` routes an installed bridgegen's
``_Machine._generic`` to this backend.  Device-resident API: ``contract``.
Multi-GPU: ``shard``.  Kernels: libbgx.so (C ABI in include/bgx.h).
"""

from . import einsum, interp  # noqa: F401
from .api import contract, contract_host  # noqa: F401
from .prepared import Prepared, prepare  # noqa: F401
from .schedule import Schedule  # noqa: F401
from .einsum import (BF16, F16, F32, F64, EinsumError, EinsumSpec,  # noqa: F401
                     build_einsum_function, derive_maps, parse_einsum)
from .interp import (DEFAULT_STEP_LIMIT, InterpError, StepLimitExceeded,  # noqa: F401
                     TensorValue, run_function)

__version__ = "0.1.0"
