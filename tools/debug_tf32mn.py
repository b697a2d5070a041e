import ctypes as C, sys, itertools
import torch
sys.path.insert(0, ".")
exec(open("tools/debug_gemm.py").read().split("for elem in")[0])
L.moses_debug_set_mn.argtypes = [C.c_int] * 5
for swz, lay, sbo in itertools.product((3, 4, 5, 6), (2, 1), (512, 1024)):
    L.moses_debug_set_mn(1, swz, lay, sbo, 1024)
    print("swz", swz, "layout", lay, "sbo", sbo)
    case(4, 128, 64, 128, 0, 1, 64)
    case(4, 128, 128, 128, 1, 1, 128)
