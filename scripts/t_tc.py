import numpy as np, sys
sys.path.insert(0,'.')
from tests.test_gpu_units import dcontract, rand, close
rng=np.random.default_rng(0)
for xs, ash in [((4,3,2,5,6,7),(2,9,5,3,8)), ((1,3,2,5,6,7),(2,9,5,3,8)), ((4,3,2,5,6,7),(2,4,5,3,8)), ((1,3,2,5,6,7),(2,4,5,3,8)), ((4,3,2,5,6,7),(2,9,5,3,1))]:
    X1=rand(rng,xs); A=rand(rng,ash)
    out,ref=dcontract(X1,"xabdDf",A,"sudar","xbDfsur",gemm=2)
    err=np.abs(out-ref); bad=np.argwhere(err>1e-3*np.abs(ref).max())
    print(xs, ash, close(out,ref), len(bad), "of", out.size, bad[:2].tolist())
