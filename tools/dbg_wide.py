import numpy as np, sys, os
sys.path.insert(0, '/root/repo')
import oracle, paper_2406_17981_b200 as T
from oracle import rel_l2
O = oracle.Oracle()
for levels in ([64,64,64], [64,16,16], [16,64,16], [64,64,16], [32,64,64]):
    s = int(np.prod(levels))
    x = O.random_vector([3]+levels, 2, 0.5)
    xs = [x[i*s:(i+1)*s] for i in range(3)]
    ys = np.concatenate(O.dyadic_apply(levels, xs, mode="signs"))
    for prec in (T.C128, T.C64):
        op = T.Operator.split_ex(T.BlockGenerator.dyadic(levels), precision=prec)
        y = op.apply(x)
        errs = [rel_l2(y[i*s:(i+1)*s], ys[i*s:(i+1)*s]) for i in range(3)]
        print(levels, prec, ["%.2e" % e for e in errs], os.environ.get("TSK_NO_WIDE"))
