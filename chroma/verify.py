"""Drop-in module path: `chroma.verify` -> paper_2107_00075_b200.verify (the B200 backend).

Reference: /root/reference/pkg/src/chroma/verify.py.  Existing code that imports the
reference package keeps working unchanged with this repository on its path."""
from paper_2107_00075_b200 import verify as _impl
from paper_2107_00075_b200.verify import *  # noqa: F401,F403

__all__ = list(getattr(_impl, "__all__", []))


def __getattr__(name):
    return getattr(_impl, name)
