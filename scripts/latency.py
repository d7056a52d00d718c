"""Dependent-op latencies on the device (bcs_selftest 40..44)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import _native
lib = _native.lib()
r = ctypes.c_ulonglong()
for what, name in [(40, "dadd"), (41, "dmul"), (42, "dfma"), (43, "shfl f64"), (44, "shfl b32")]:
    n = 4096
    lib.bcs_selftest(what, n, 0, ctypes.byref(r))
    lib.bcs_selftest(what, n, 0, ctypes.byref(r))
    print(f"{name:10s} {r.value / n:.2f} cycles/op")
