"""B200-native CKKS evaluation engine with the module API of ``rnscope``.

Submodules mirror the reference package: ``rns``, ``transform``, ``baseconv``,
``keyswitch``, ``params``, ``vectors``, ``instrument``; ``ckks`` adds
encode/decode, hmult+relinearize, rescale and hrot on top.  Arithmetic runs in
csrc/libckks_b200.so (hand-written sm_100a CUDA behind a C ABI,
include/ckks_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"
