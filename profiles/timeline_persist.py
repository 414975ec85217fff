import sys
sys.path.insert(0,'profiles')
from timeline_summary import load_runs
import numpy as np
for f in sys.argv[1:]:
    r=np.array(load_runs(f)[-1],dtype=np.int64)
    s,e,fi=r[:,1],r[:,2],r[:,3]
    ps=(e-s)/1e3; red=(fi-e)/1e3; g=(s[1:]-fi[:-1])/1e3
    print(f, "pass even %.1f odd %.1f | reduce %.1f | vbuild %.1f | total %.2f ms" % (np.median(ps[0::2]), np.median(ps[1::2]), np.median(red), np.median(g), (fi[-1]-s[0])/1e6))
