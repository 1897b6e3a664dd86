"""B200-native server-side hot path of arXiv 2103.05875 light-probe streaming.

Drop-in for the reference's probe-update, change-selection and packing
entry points (``probestream.{volume,selection,packing}``), backed by
hand-written sm_100a CUDA kernels behind the C ABI in
``include/probestream.h``.  See DESIGN.md.
"""

from .errors import LayoutMismatchError, NativeLibraryError, SlotOverflowError
from .volume import (
    AtlasKind,
    ProbeAtlas,
    ProbeVolume,
    oct_decode,
    oct_encode,
    raw_bits,
    throughput_bps,
)

__all__ = [
    "AtlasKind",
    "ProbeAtlas",
    "ProbeVolume",
    "oct_decode",
    "oct_encode",
    "raw_bits",
    "throughput_bps",
    "LayoutMismatchError",
    "SlotOverflowError",
    "NativeLibraryError",
]

__version__ = "0.1.0"
