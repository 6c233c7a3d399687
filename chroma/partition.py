"""Drop-in module path: `chroma.partition` -> paper_2107_00075_b200.partition (the B200 backend).

Reference: /root/reference/pkg/src/chroma/partition.py.  Existing code that imports the
reference package keeps working unchanged with this repository on its path."""
from paper_2107_00075_b200 import partition as _impl
from paper_2107_00075_b200.partition import *  # noqa: F401,F403

__all__ = list(getattr(_impl, "__all__", []))


def __getattr__(name):
    return getattr(_impl, name)
