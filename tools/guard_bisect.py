"""Find the first native call after which a COMPUTED NaN (any NaN whose bits differ from the
Guards poison pattern) appears in a guarded allocation.  Debug tool for tests/test_gpu_guards.py.

    python tools/guard_bisect.py d m decades rel
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import _native as N  # noqa: E402

d, m, decades, rel = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), float(sys.argv[4])
rng = np.random.default_rng(m)
q1, _ = np.linalg.qr(rng.standard_normal((d, m)))
q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
sig = 10.0 ** (-decades * np.arange(m) / max(m - 1, 1))
vals = np.asfortranarray((q1 * sig) @ q2.T)

D.Guards.enable()
seen = set()
orig_check = N.check
calls = [0]


def scan(what):
    torch.cuda.synchronize()
    for k, (raw, nbytes) in enumerate(list(D.Guards._live)):
        if k in seen:
            continue
        pay = raw[D.Guards.ZONE // 8: (D.Guards.ZONE + nbytes) // 8]
        f = pay.view(torch.float64)
        bad = torch.isnan(f) & (pay != D.Guards.POISON)
        nb = int(bad.sum())
        if nb:
            idx = torch.nonzero(bad).flatten()[:8].tolist()
            npoison = int((pay == D.Guards.POISON).sum())
            print(f"[bisect] after call #{calls[0]} '{what}': allocation {k} ({nbytes} bytes) has {nb} computed NaNs, "
                  f"first at elements {idx}; {npoison} poison words remain", flush=True)
            seen.add(k)


def check(rc, what="native call"):
    orig_check(rc, what)
    calls[0] += 1
    scan(what)


N.check = check
D.N.check = check
out = H.pod(H.SnapshotBlock(H.InnerProductSpace(d), vals), rel * float(np.linalg.norm(vals)), want_right=True)
modes = np.asarray(out.modes)
print("modes NaN count", int(np.isnan(modes).sum()), "of", modes.size, "; columns with NaN:",
      np.nonzero(np.isnan(modes).any(axis=0))[0][:10])
print("guards checked:", D.Guards.check())
nanpos = np.argwhere(np.isnan(modes))
rows = np.unique(nanpos[:, 0])
cols = np.unique(nanpos[:, 1])
print("NaN rows:", rows[:40], "... count", rows.size, "; NaN cols:", cols[:40], "... count", cols.size)
bits = modes.view(np.int64)[np.isnan(modes)]
print("poison words among them:", int((bits == D.Guards.POISON).sum()), "of", bits.size)
if out.right is not None:
    r = np.asarray(out.right)
    print("right factor NaNs:", int(np.isnan(r).sum()), "of", r.size)
