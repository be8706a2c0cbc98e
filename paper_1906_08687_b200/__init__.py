"""paper_1906_08687_b200 — B200-native (sm_100a) hot path of LMFAO (arXiv 1906.08687).

Evaluates batches of group-by aggregates whose UDAFs are sums of products of
per-attribute functions over the natural join of an acyclic schema, bottom-up
over a join tree, without materialising the join.  The work runs in the CUDA
kernels of liblmfao_gpu.so behind the C ABI include/lmfao_gpu.h; `lmfao` is the
thin ctypes binding.
"""
__all__ = ["lmfao"]
