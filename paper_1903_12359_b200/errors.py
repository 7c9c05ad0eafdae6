"""Exception classes of the reference API (same names and bases).

mesh.py:15 MeshError(ValueError), flatten.py:24 SolveError(RuntimeError),
welding.py:35 WeldError(RuntimeError), partition.py:21 PartitionError(ValueError),
pipeline.py:32 ValidationError(ValueError).
"""


class MeshError(ValueError):
    """Raised for invalid mesh data (bad indices, degenerate or non-manifold input)."""


class SolveError(RuntimeError):
    """Raised when a sparse solve fails or violates its residual contract."""


class WeldError(RuntimeError):
    """Raised when welding preconditions or numerical guards fail."""


class PartitionError(ValueError):
    """Raised for invalid cut sets or unweldable partitions."""


class ValidationError(ValueError):
    """Configuration or input-topology mismatch."""
