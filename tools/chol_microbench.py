import ctypes, sys
sys.path.insert(0, '.')
lib = ctypes.CDLL('paper_2409_12190_b200/libbae_b200.so')
out = (ctypes.c_longlong * 4)()
print(lib.bae_dev_chol_microbench(20, out), 'potrf_inv48 gemm48 chol16+inv chol16 (cycles):', list(out))
