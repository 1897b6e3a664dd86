"""Exception classes of the reference, re-declared for the drop-in.

``LayoutMismatchError`` mirrors ``probestream.selection.LayoutMismatchError``
(selection.py:25-26) and ``SlotOverflowError`` mirrors
``probestream.packing.SlotOverflowError`` (packing.py:227-228); both keep the
reference's base classes so ``except ValueError`` / ``except RuntimeError``
callers behave identically.
"""


class LayoutMismatchError(ValueError):
    pass


class SlotOverflowError(RuntimeError):
    pass


class NativeLibraryError(ImportError):
    """The CUDA extension is missing or was built for another ABI."""
