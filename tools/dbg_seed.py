import sys, os
sys.path.insert(0,'.')
import numpy as np, importlib.util
spec=importlib.util.spec_from_file_location('sc','tools/stress_class.py'); sc=importlib.util.module_from_spec(spec); spec.loader.exec_module(sc)
from paper_1509_01506_b200 import _native
from oracle import oracle as O
seed=int(sys.argv[1]); n=int(sys.argv[2])
rng=np.random.default_rng(seed)
lb=int(rng.choice([1,2,3,4,4,5,6])); os.environ["KS_TILE_LB"]=os.environ.get("FORCE_LB", str(lb))
kind,dfa=sc.random_dfa(rng)
codes=np.random.default_rng(1).integers(0,4,n).astype(np.uint8)
want=O.ref_sequential_count(dfa,codes)[0]
c=_native.DeviceContext(0); dh=c.dfa(dfa); sh=c.upload_codes(codes)
print(dh.info)
for i in range(4):
    got=c.count(dh,sh)
    d=got-want
    print("call",i,"equal",bool((d==0).all()),"nonzero diffs",int((d!=0).sum()),"sum diff",int(d.sum()), "total", int(want.sum()), c.stats(), flush=True)
