"""Exception types of the assembly boundary.

The hierarchy is the reference's (``/root/reference/pkg/src/nlfem/errors.py:4-13``):

* :class:`ConfigurationError` (a ``ValueError``) -- invalid inputs, raised
  before any device work;
* :class:`NumericalError` (a ``RuntimeError``) -- a nonfinite local
  contribution, naming the element pair;
* :class:`MeshFormatError` (a ``ConfigurationError``) -- malformed mesh text.

When the reference package is importable (``nlfem.errors``), each class here
also *subclasses* the reference's class of the same name, so a caller that
swapped only the assembly import keeps catching ``nlfem.errors.*``.
Without it the classes stand alone with the same bases and names.

:class:`DeviceError` is this package's own: the CUDA library is missing, no
GPU is visible, or a launch failed (there is no CPU fallback).
"""

import importlib


def _reference_errors():
    try:
        return importlib.import_module("nlfem.errors")
    except Exception:  # noqa: BLE001 -- absent (or broken) reference: stand-alone hierarchy
        return None


_REF = _reference_errors()


def _bases(name, *own):
    ref = getattr(_REF, name, None) if _REF is not None else None
    if ref is None:
        return own
    return tuple(b for b in own if not issubclass(ref, b)) + (ref,)


class ConfigurationError(*_bases("ConfigurationError", ValueError)):
    """Inputs that cannot be assembled (bad shapes, unknown options, ...)."""


class NumericalError(*_bases("NumericalError", RuntimeError)):
    """A local contribution evaluated to inf or nan."""


class MeshFormatError(*_bases("MeshFormatError", ConfigurationError)):
    """A mesh or matrix text file that does not parse."""


class DeviceError(RuntimeError):
    """The CUDA library is missing, no B200 is visible, or a launch failed.

    There is no CPU fallback: the product path raises this instead.
    """


REFERENCE_LINKED = _REF is not None
