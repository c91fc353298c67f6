"""solve_timeline.py against another build of the library: python tools/solve_timeline_lib.py LIB CONFIG N"""
import ctypes as C, os, sys, runpy
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_05460_b200 as afn
lib = C.CDLL(os.path.abspath(sys.argv[1]))
for name, (res, args) in afn._sig.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
afn._lib = lib
sys.argv = [sys.argv[0]] + sys.argv[2:]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "solve_timeline.py"), run_name="__main__")
