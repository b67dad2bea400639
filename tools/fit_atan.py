import numpy as np
from scipy.optimize import linprog
def fit(nc, scale=2.0):
    # minimax via LP on a dense grid: min e s.t. |scale*atan(q) - q*P(q^2)| <= e
    q = np.linspace(0, 1, 4000)
    A = np.stack([q * q**(2*i) for i in range(nc)], 1)
    f = scale*np.arctan(q)
    # vars: c (nc), e
    Aub = np.vstack([np.hstack([A, -np.ones((len(q),1))]), np.hstack([-A, -np.ones((len(q),1))])])
    bub = np.concatenate([f, -f])
    res = linprog(np.r_[np.zeros(nc), 1], A_ub=Aub, b_ub=bub, bounds=[(None,None)]*nc+[(0,None)], method="highs")
    return res.x[:nc], res.x[nc]
for nc in (6,7,8):
    c, e = fit(nc)
    # fp32 horner evaluation error
    q = np.linspace(-1, 1, 200001).astype(np.float32)
    s = (q*q).astype(np.float32)
    p = np.float32(c[-1])
    for ci in c[-2::-1]:
        p = (p*s + np.float32(ci)).astype(np.float32)
    t = (q*p).astype(np.float32)
    err = np.abs(t.astype(np.float64) - 2*np.arctan(q.astype(np.float64))).max()
    print(nc, "minimax", e, "fp32 eval", err, repr([float(np.float32(x)) for x in c]))
