import ctypes, sys
sys.path.insert(0, '.')
lib = ctypes.CDLL('paper_2409_12190_b200/libbae_b200.so')
out = (ctypes.c_longlong * 3)()
print(lib.bae_dev_chol_microbench(20, out), list(out))
