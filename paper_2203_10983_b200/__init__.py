"""B200-native BNS-GCN hot path (arXiv 2203.10983): C-ABI library libbns.so + thin ctypes binding.

The product path is ``paper_2203_10983_b200.bns`` (the binding) over ``libbns.so`` (csrc/).  ``inputs`` holds the
seeded workload generators (setup only).
"""
