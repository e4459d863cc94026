"""Device-resident result fields that become numpy arrays on their first host read.

The estimators' posterior statistics (fastfca.py:466, fca.py:211) are computed on the device at
the end of a run.  They are kept there -- a device consumer (the Wiener images) uses them in
place -- and a field is copied to the host once, the first time Python code reads it.  To the
caller the dataclass fields are ordinary numpy arrays (attribute access, ``dataclasses.replace /
asdict``, equality, repr and pickling all see numpy).
"""

from __future__ import annotations

import numpy as np


class DeviceArray:
    """A device-resident array (a torch CUDA tensor) copied to numpy on first host access."""

    __slots__ = ("t",)

    def __init__(self, t):
        self.t = t

    def numpy(self) -> np.ndarray:
        return self.t.cpu().numpy()


class LazyHostFields:
    """Mixin for dataclasses whose fields in ``_LAZY`` may hold a ``DeviceArray``."""

    _LAZY: tuple = ()

    def __getattribute__(self, name):
        if name in type(self)._LAZY:
            d = object.__getattribute__(self, "__dict__")
            val = d[name]
            if isinstance(val, DeviceArray):
                val = d[name] = val.numpy()
            return val
        return object.__getattribute__(self, name)

    def __getstate__(self):
        d = dict(object.__getattribute__(self, "__dict__"))
        for k in type(self)._LAZY:
            d[k] = getattr(self, k)
        return d

    def device_tensor(self, name: str):
        """The field as a device tensor while it has not been copied to the host, else None."""
        val = object.__getattribute__(self, "__dict__")[name]
        return val.t if isinstance(val, DeviceArray) else None
