"""eqc -- B200-native sort-last image compositing and RLE frame transport.

The hot path of Eilemann's parallel rendering thesis (arxiv 1902.08755):
depth compositing, ordered alpha blending, per-component RLE with the
bit-swizzle preconditioner, and the direct-send / binary-swap multi-GPU
schedules, as hand-written sm_100a CUDA kernels behind the C ABI of
``include/eqc.h`` (``libeqc.so``).

    from paper_1902_08755_b200 import eqc     # ctypes binding; raises if libeqc.so is missing
    python -m paper_1902_08755_b200.build     # nvcc -> libeqc.so (sm_100a)
"""
