import sys, numpy as np
sys.path.insert(0, '.')
import paper_2402_04403_b200 as gb
d = np.load('tests/golden/golden.npz')
name = sys.argv[1]
c = {k.split('/', 1)[1]: d[k] for k in d.files if k.startswith(name + '/')}
el = gb.EdgeList(n=int(c['n']), src=c['src'], dst=c['dst'], w=c['w'], directed=bool(c['directed']))
y = gb.LabelVector(labels=c['labels'], k=int(c['k']))
z = gb.embed_serial(el, y, variant="pull")
print(name, float(np.max(np.abs(z - c['z_serial']))), flush=True)
