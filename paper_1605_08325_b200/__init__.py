"""B200-native parameter exchange of Theano-MPI (arXiv 1605.08325): AR, ASA, ASA16, EASGD.

The compute path is libtm.so (hand-written sm_100a CUDA behind the C ABI in
include/tm.h); `paper_1605_08325_b200.tm` is its thin ctypes binding.
"""
