"""B200-native GLoP matching path (arXiv 1704.02278): PFAC over 8-byte
prefixes and chunk-parallel KMP as sm_100a kernels behind a C ABI
(include/glop.h), with the reference's C++ API kept in include/logtrawl/.

Python entry points live in `paper_1704_02278_b200.glop` (ctypes binding) and
`paper_1704_02278_b200.shards` (multi-GPU sharding over torch.distributed).
"""
__all__ = ["glop"]
