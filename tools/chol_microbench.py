import ctypes, sys
sys.path.insert(0, '.')
lib = ctypes.CDLL('paper_2409_12190_b200/libbae_b200.so')
out = (ctypes.c_longlong * 40)()
print(lib.bae_dev_chol_microbench(20, out), 'potrf_inv48 gemm48 chol16+inv chol16 (cycles):', list(out)[:4])
st = [x for x in list(out)[8:28] if x]
print('potrf phases (cycles since the previous barrier):', [b - a for a, b in zip(st, st[1:])])
