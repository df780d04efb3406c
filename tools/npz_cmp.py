"""Max normwise difference of every array of two npz files (development aid)."""
import sys
import numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    x, y = a[k].astype(np.float64), b[k].astype(np.float64)
    print(f"{k:10s} max|a-b| / max|a| = {np.abs(x - y).max() / max(np.abs(x).max(), 1e-300):.3e}  equal={np.array_equal(x, y)}")
