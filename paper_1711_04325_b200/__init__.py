"""B200-native gradient exchange + blended RMSprop/SGD update of arXiv 1711.04325.

The product is ``liblmsgd.so`` (C ABI in ``include/lmsgd.h``, sm_100a kernels in
``csrc/``); ``lmsgd`` is its thin ctypes binding.  Importing this package loads
the library and fails loudly if it has not been built -- there is no CPU path.
"""
from .lmsgd import *  # noqa: F401,F403
from .lmsgd import LIB_PATH, EXPORTED, LmsgdError, Context, lib  # noqa: F401
from .optim import LMSGD, BucketedLMSGD  # noqa: F401,E402
