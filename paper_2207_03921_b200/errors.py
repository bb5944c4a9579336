"""Exception types of the assembly boundary.

Same hierarchy as the reference (``/root/reference/pkg/src/nlfem/errors.py:4-13``)
so callers catching the reference's exceptions keep working:

* :class:`ConfigurationError` -- invalid inputs, raised before any device work;
* :class:`NumericalError` -- a nonfinite local contribution, naming the pair;
* :class:`MeshFormatError` -- malformed mesh text (a configuration error).
"""


class ConfigurationError(ValueError):
    """Inputs that cannot be assembled (bad shapes, unknown options, ...)."""


class NumericalError(RuntimeError):
    """A local contribution evaluated to inf or nan."""


class MeshFormatError(ConfigurationError):
    """A mesh or matrix text file that does not parse."""


class DeviceError(RuntimeError):
    """The CUDA library is missing, no B200 is visible, or a launch failed.

    There is no CPU fallback: the product path raises this instead.
    """
