import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import _native
L = _native.lib()
r = ctypes.c_ulonglong()
for variant in (0, 1):
    for warps in (8, 64, 512, 4096):
        steps = 20000
        L.bcs_selftest(30 + variant, steps, warps, ctypes.byref(r))
        print(f"variant {variant} warps {warps:5d}: {r.value / steps:8.1f} ns per hop", flush=True)
