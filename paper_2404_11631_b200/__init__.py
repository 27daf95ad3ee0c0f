"""B200-native (sm_100a) hot path of the arXiv 2404.11631 simulation-optimization
benchmark: a drop-in "cuda" backend and device-resident problem adapters for the
reference package's (sobench) Python solver API.  See DESIGN.md.
"""
from .backend import CudaBackend, make_backend
from .errors import (ConfigurationError, DegeneratePair, DeviceError, DimensionMismatch,
                     EmptyRequest, InsufficientSamples, InvalidConstraint, InvalidGradient,
                     RunAborted, SobenchError, SolverStall, UndefinedMetric)
from .sampling import (GaussianSpec, RngStream, sample_returns, sample_returns_device,
                       standard_normal, standard_normal_device, uniform01, uniform01_device)

__version__ = "0.1.0"
