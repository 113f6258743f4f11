"""Long rows per SELL matrix of an engine (V^T, [U | Ahat], U^T,
[Ahat^T | V]) above 16 / 32 / 64 / 128 / 256 entries, with the row count and
the longest row, for the corpus and configs 2 / 4 (one board): the data behind
the adaptive long-row threshold (kr_engine.cu, kLongRowBudget)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sps  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402


def mat(t, shape):
    ptr, idx, val = t
    n = len(ptr) - 1
    if n == shape[1]: return sps.csc_matrix((val, idx, ptr), shape=shape)
    return sps.csr_matrix((val, idx, ptr), shape=shape)
def cnt(name, kw):
    p=H.builtin(name,**kw); f=p.sparsify("b",True); fa=f.factors()
    R,C,K=p.rows,p.cols,f.k
    A=mat(fa['ahat'],(R,C)).tocsr(); U=mat(fa['u'],(R,K)).tocsr(); V=mat(fa['v'],(C,K)).tocsr()
    lens={'VT':np.diff(V.tocsc().indptr),'UA':np.diff(U.indptr)+np.diff(A.indptr),'UT':np.diff(U.tocsc().indptr),'AV':np.diff(A.tocsc().indptr)+np.diff(V.indptr)}
    out={}
    for k,l in lens.items():
        out[k]=[int((l>T).sum()) for T in (16,32,64,128,256)]+[len(l), int(l.max())]
    print(name, out)
cnt("twenty_card",{}); cnt("bench",dict(seed=2,hands=100)); cnt("golden",{})
cnt("river_full",dict(seed=1, board="Kc9d7c4d2c", deck=26, tree=3))
cnt("river_full",dict(seed=1, board="Ks7d4c2h9s", tree=3))
