import ctypes, sys
sys.path.insert(0, '.')
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import _lib
rt = gpb.start_runtime()
lib = _lib.load()
for sec in (0.05, 0.05, 1.0, 3.0):
    out = ctypes.c_double()
    _lib.check(lib.gpb_int8_peak_probe(rt.handle, sec, ctypes.byref(out)))
    print(f"int8 tcgen05 probe ({sec} s): {out.value:.1f} TOPS", flush=True)
out = ctypes.c_double()
_lib.check(lib.gpb_fp64_peak_probe(rt.handle, 1.0, ctypes.byref(out)))
print("fp64", out.value)
rt.stop()
