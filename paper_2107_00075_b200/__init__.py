"""B200-native distributed speculate-and-iterate graph colouring (arXiv 2107.00075).

Drop-in for the reference package ``chroma``: the modules graph, partition,
runtime, localcolor, protocol and verify keep the reference's names, arguments and
error behaviour, while the colouring path runs in libchroma_b200.so (hand-written
sm_100a CUDA behind a C ABI, NCCL over NVLink for multi-GPU).
"""
from . import graph, localcolor, partition, protocol, runtime, verify  # noqa: F401
from ._lib import launch_count, lib, set_device  # noqa: F401

__all__ = ["graph", "partition", "runtime", "localcolor", "protocol", "verify", "lib",
           "launch_count", "set_device"]
