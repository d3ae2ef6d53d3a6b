"""B200-native windowed root-MUSIC BOS fringe demodulation (arxiv 1910.11872).

The product is ``libbosrm.so`` (hand-written sm_100a CUDA behind the C ABI declared in
``include/bos_rootmusic.h``); :mod:`.bosrm` is the thin ctypes binding with the same names.
"""

__all__ = ["bosrm", "synth", "sharding"]
