"""B200-native block-preconditioned GMRES for mixed virtual elements (arXiv 1901.02330).

The product path is libvem_mixed.so (sm_100a CUDA, C ABI in include/vem_mixed.h)
driven through the thin ctypes binding below.  No CPU fallback exists.
"""
from .binding import (PRECOND_BLOCK_REG, PRECOND_BLOCK_REG_M, PRECOND_BLOCK_SCHUR, PRECOND_BLOCK_SCHUR_AMG, PRECOND_BLOCK_SCHUR_AMG_F32, PRECOND_NONE, EXPORTS, LIB_PATH,  # noqa: F401
                      Assembled, VemError, VemMixed, default_options, load_library)
