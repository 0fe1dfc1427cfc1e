import sys, numpy as np
sys.path.insert(0, '.')
import paper_2402_04403_b200 as gb
d = np.load('tests/golden/golden.npz')
names = sorted({k.split('/')[0] for k in d.files if k.endswith('/z_serial')})
for name in names:
    c = {k.split('/', 1)[1]: d[k] for k in d.files if k.startswith(name + '/')}
    el = gb.EdgeList(n=int(c['n']), src=c['src'], dst=c['dst'], w=c['w'], directed=bool(c['directed']))
    y = gb.LabelVector(labels=c['labels'], k=int(c['k']))
    z = gb.embed_serial(el, y, variant="pull")
    w4 = (__import__("ctypes").c_uint * 4)(); __import__("paper_2402_04403_b200")._lib.lib.gee_debug_word(__import__("ctypes").byref(w4)); print(" dbg", list(w4))
    print(name, float(np.max(np.abs(z - c['z_serial']))), flush=True)
import ctypes
from paper_2402_04403_b200 import _lib
w = (ctypes.c_uint * 4)()
_lib.lib.gee_debug_word(ctypes.byref(w))
print("debug word", list(w))
