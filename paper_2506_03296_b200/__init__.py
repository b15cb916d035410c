"""B200-native (sm_100a) decode-attention hot path of APEX (arXiv 2506.03296).

C ABI: include/apex.h (libapex.so).  Python: ``apex`` (ctypes mirror of the ABI),
``kvcache.PagedKVCache`` (torch-owned memory + handle), ``sharding`` (request /
KV-head partitioning across ranks).  No CPU fallback exists.
"""
__all__ = ["apex", "kvcache", "sharding"]
