"""paper_1611_06945_b200 — B200-native convolution hot path of Boda (arXiv:1611.06945).

A from-scratch sm_100a implementation of the reference package ``cuclgen``'s
conv path (AlexNet / NiN / GoogLeNet conv ops, bias + ReLU epilogue, autotuned
variant choice), kept behind the reference's op-description and
variant/tuning API:

* ``frontend``  ConvParams / OpNode / conv_graph / flops_of    (cuclgen/frontend.py)
* ``ndarray``   DimsSpec / NdArray / convert_format              (cuclgen/ndarray.py)
* ``corpus``    the 43-op Appendix-A corpus, BenchOp, CSV I/O     (cuclgen/corpus.py)
* ``variants``  TuneParams / Variant / VARIANTS / select_variant (cuclgen/variants.py)
* ``tuner``     op_signature / sweep / TuneDB (on-device timing)  (cuclgen/tuner.py)
* ``runner``    execute_node / node_test_inputs                   (cuclgen/runner.py)
* ``backend``   ctypes binding of libb2conv.so (include/b2conv.h) (cuclgen/backend.py:1104 run_kernel)

The kernels live in ``csrc/`` and are built in-tree into ``libb2conv.so``.
There is no CPU fallback: executing without the library (or without a GPU)
raises.
"""

__version__ = "0.1.0"

from .errors import CuclgenError

__all__ = ["CuclgenError", "__version__"]
