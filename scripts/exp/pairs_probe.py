import ctypes, os
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpairs_probe.so"))
lib.pairs_probe(0)
