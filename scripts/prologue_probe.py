import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2412_08264_b200 import batched, bilevel
orig = batched.recycle_update_native
L = None
stats = []
def wrapped(*a, **k):
    from paper_2412_08264_b200 import _lib
    lib = _lib.lib()
    fn = lib.kr_recycle_update
    t0 = time.perf_counter()
    marks = {}
    class Proxy:
        def __getattr__(self, name):
            f = getattr(lib, name)
            if name == "kr_recycle_update":
                def g(*aa):
                    marks["call"] = time.perf_counter()
                    r = f(*aa)
                    marks["ret"] = time.perf_counter()
                    return r
                return g
            return f
    old = _lib.lib
    _lib.lib = lambda: Proxy()
    try:
        r = orig(*a, **k)
    finally:
        _lib.lib = old
    t1 = time.perf_counter()
    if "call" in marks:
        stats.append(((marks["call"] - t0) * 1e3, (t1 - marks["ret"]) * 1e3))
    return r
bilevel.recycle_update_native = wrapped
sys.argv = ["host_marks"]
exec(open("/root/repo/scripts/host_marks.py").read().replace("wrap(batched, \"recycle_update_native\", \"native\")", "").replace("bilevel.recycle_update_native = batched.recycle_update_native", ""))
print("prologue/epilogue ms per call (last 8):", [(round(a, 3), round(b, 3)) for a, b in stats[-8:]])
