"""Reproducer of the r2f failure (one LBR round-trip case with a -0.0 / 1e-10 price):
the same row through batch_price -> batch_iv and the fused price_iv, three times, and
the LBR call on literal -0.0 / +0.0 prices (profiles/README.md, r2f)."""
import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, paper_2604_27210_b200 as fv
a={'model': 'black', 'flag': -1.0, 'underlying': 2.279255594198151e+122, 'strike': 7.81815240030788e+117, 't': 3.279971536884726e-05, 'r': 0.026461581327708927, 'q': 0.0, 'sigma': 1.9518652727891157e-10}
base=(["p"],[a['underlying']],[a['strike']],[a['t']],[a['r']])
for rep in range(3):
    p=fv.batch_price('black',*base,[0.0],sigma=[a['sigma']])['price']
    for m in ('lbr','halley'):
        tb=fv.batch_iv('black',m,*base,price=p,q=[0.0])
        tf=fv.price_iv('black',m,*base,[0.0],sigma=[a['sigma']])
        print(rep, m, 'price', repr(p[0]), 'two-call', tb['status'][0], repr(tb['iv'][0]), '| fused', tf['status'][0], repr(tf['iv'][0]))
    tb=fv.batch_iv('black','lbr',*base,price=np.array([-0.0]),q=[0.0]); print(' lbr -0.0 literal', tb['status'][0], tb['iv'][0])
    tb=fv.batch_iv('black','lbr',*base,price=np.array([0.0]),q=[0.0]); print(' lbr +0.0 literal', tb['status'][0], tb['iv'][0])
