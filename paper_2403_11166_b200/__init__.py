"""B200-native engine for Pencil's (arXiv 2403.11166) HE linear-layer protocol.

Hot path (BASELINE.json north_star): RNS-BFV encrypt -> ciphertext x
plaintext multiply-accumulate in the NTT domain (FC / conv packings) ->
masking -> decrypt-to-additive-share, plus share arithmetic mod 2^ell, all as
hand-written sm_100a CUDA kernels behind the C ABI in include/pencil_b200.h.
"""

from .errors import (  # noqa: F401
    BankError,
    DesyncError,
    DeviceError,
    EncodeRangeError,
    FormError,
    GeometryError,
    HandshakeError,
    ParamsError,
    PencilError,
    ScaleError,
    ShapeError,
)
from .params import BfvParams  # noqa: F401

__version__ = "0.1.0"
