"""Fixtures of the `.hpd` container written by the UNMODIFIED reference writer
(hapod.io.write_matrix / write_floats, /root/reference/pkg/src/hapod/io.py:38-51, 128-133).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_hpd_golden.py

Writes tests/golden/hpd_plain.hpd, hpd_weighted.hpd, hpd_sigmas.txt; the inputs are rebuilt
by ``hpd_inputs()`` in tests/test_hpd.py (same formula)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("HAPOD_REF_SRC", "/root/reference/pkg/src"))
from hapod import io as hio  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def hpd_inputs():
    a = np.arange(35, dtype=np.float64).reshape(7, 5) / 7.0 - 2.0
    a[0, 0] = -0.0
    a[3, 2] = 1e-310           # subnormal
    a[6, 4] = -1.7976931348623157e308
    w = np.linspace(0.5, 2.0, 7)
    s = np.array([3.0, 1.0 / 3.0, 1e-300, 2.0 ** -1074, 0.1])
    return a, w, s


if __name__ == "__main__":
    a, w, s = hpd_inputs()
    hio.write_matrix(os.path.join(HERE, "hpd_plain.hpd"), a)
    hio.write_matrix(os.path.join(HERE, "hpd_weighted.hpd"), a, w)
    hio.write_floats(os.path.join(HERE, "hpd_sigmas.txt"), s)
    print("wrote hpd fixtures")
