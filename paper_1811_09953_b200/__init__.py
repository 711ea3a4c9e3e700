"""B200-native homomorphic evaluation path of Faster CryptoNets (arXiv 1811.09953).

Drop-in for the reference package's ring / fv / engine evaluation API:
Python host code (this package) over the C ABI of libfcn.so
(include/fcn.h), whose hand-written sm_100a kernels hold every ciphertext
in HBM.  There is no CPU fallback: compute calls fail loudly without a
CUDA device and the built library.
"""

__version__ = "0.1.0"
