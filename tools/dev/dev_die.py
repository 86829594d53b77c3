import ctypes, sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1611_07819_b200 import _lib as L
lib = L.load()
m = (ctypes.c_uint64 * 3)(); d0 = ctypes.c_int32(); n = ctypes.c_int32(); dm = ctypes.c_int32()
L.check(lib.gm_debug_die_map(0, m, ctypes.byref(d0), ctypes.byref(n), ctypes.byref(dm)))
bits = "".join("1" if (m[s // 64] >> (s % 64)) & 1 else "0" for s in range(n.value))
print("die0_sms", d0.value, "sms", n.value, "max_sig_distance", dm.value)
print("die-1 SMs by smid:", bits)
