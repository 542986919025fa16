"""B200-native edge-alignment detector: the reference `edgealign` search path
(arxiv 2112.05576) as hand-written sm_100a kernels behind a C-ABI
(include/edgealign_b200.h), with a Python mirror of the reference API.

Importing is cheap and device-free; the first compute call loads
libedgealign_b200.so and fails loudly if it is missing or no GPU is present.
"""
from . import abi, errors  # noqa: F401
from .abi import *  # noqa: F401,F403
from .api import *  # noqa: F401,F403
from .errors import (BoundsError, BudgetError, CudaError, EmptyModelError, Error,  # noqa: F401
                     GeometryError, InvalidArgument, ParseError, SizeError)
