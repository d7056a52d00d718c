import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07882_b200 import _native
L = _native.lib()
n = 20000
for mode, name in enumerate(["relaxed", "relaxed+fence", "atomicExch", "volatile", "release/acquire"]):
    r = ctypes.c_ulonglong()
    st = L.bcs_selftest(10 + mode, n, 0, ctypes.byref(r))
    print(f"{name:16s} one-way hop {r.value / (2 * n):8.1f} ns  (st={st})", flush=True)
