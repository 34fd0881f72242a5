"""Print the measured SM -> die map of GPU 0 (dflow_device_die_map)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04467_b200 as D  # noqa: E402

n = 148
arr = (C.c_int32 * n)()
a = C.c_double(0)
st = D.dflow_device_die_map(0, arr, n, C.byref(a))
print("status", D.STATUS.get(st), (D.dflow_last_error() or b"").decode(), "agreement", a.value)
print("die0", sum(1 for x in arr if x == 0), "die1", sum(1 for x in arr if x == 1))
print("".join(str(x) if x >= 0 else "?" for x in arr))
