"""B200-native hot path of the Shor simulator of arXiv 1801.01434.

Drop-in modules mirroring the reference package ``shorsim``:

* ``numtheory`` -- exact integer math (host)
* ``qstate``    -- device-resident register: modexp, collapse, Born-rule read
* ``qft``       -- the QFT engines, all served by the sm_100a direct-DFT kernel
* ``shor``      -- the end-to-end driver
* ``distributed`` -- the same pipeline sharded over ranks (torch.distributed)

The kernels live in ``libshorb200.so`` (C ABI: include/shorb200.h), built by
``paper_1801_01434_b200.build``.
"""

from . import numtheory  # noqa: F401  (pure host code, importable without a GPU)

__all__ = ["numtheory", "qstate", "qft", "shor", "distributed", "build"]
