"""Clusters of the row-mask kernel the device holds at once, per cluster size and shape (tt_rows_max_clusters)."""
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1609_04104_b200 import _lib as L
L.load()
for (n, R, S) in [(256, 16, 52), (256, 20, 64), (128, 10, 32), (1024, 32, 128)]:
    for c in (2, 4, 8, 16):
        m = C.c_int(0)
        rc = L.lib().tt_rows_max_clusters(n, n, R, S, c, C.byref(m))
        print(n, R, S, 'cluster', c, 'rc', rc, 'max clusters', m.value)
