"""GPU debug harness for the tcgen05 matmul layouts (structured inputs)."""
import numpy as np
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10855_b200 as jb

np.set_printoptions(linewidth=200, precision=3, suppress=True)
def t(x): return x.astype(np.float32)
rng = np.random.default_rng(0)
# integer-valued inputs are exact in tf32: lo = 0
n, m, l = 128, 32, 64
B = t(rng.integers(-4, 5, (m, l)))
A = np.zeros((n, m), np.float32); A[np.arange(32), np.arange(32)] = 1
C = jb.matmul(A, B)
print("case1 A=I: rows0-31 ok?", np.array_equal(C[:32], B), "rest zero?", not C[32:].any())
for i in range(4):
    row = C[i]
    # find matching B row / B col
    mr = [j for j in range(m) if np.array_equal(row[:], B[j])]
    print(" C row", i, "matches B rows", mr, "C[i,:8]", row[:8], "B[i,:8]", B[i, :8])
A = t(rng.integers(-4, 5, (n, m)))
B = np.zeros((m, l), np.float32); B[np.arange(32), np.arange(32)] = 1
C = jb.matmul(A, B)
print("case2 B=I: C[:, :32]==A?", np.array_equal(C[:, :32], A), "C[:,32:]==0?", not C[:, 32:].any())
print(" C[0,:8]", C[0, :8], "A[0,:8]", A[0, :8])
print(" C[1,:8]", C[1, :8], "A[1,:8]", A[1, :8])
print(" C[8,:8]", C[8, :8], "A[8,:8]", A[8, :8])
# single nonzero probes
for (ai, ak) in [(0, 0), (0, 1), (0, 4), (0, 8), (1, 0), (5, 3), (9, 17)]:
    A = np.zeros((n, m), np.float32); A[ai, ak] = 1
    B = np.zeros((m, l), np.float32)
    B[ak, :] = np.arange(l)
    C = jb.matmul(A, B)
    nz = np.argwhere(C != 0)
    print(f" probe A[{ai},{ak}]=1, B[{ak},:]=0..63 -> nonzero C rows {sorted(set(nz[:,0].tolist()))[:8]} first vals {C[nz[0][0], :6] if len(nz) else None}")
for (bk, bj) in [(0, 0), (0, 1), (0, 4), (1, 0), (3, 5), (0, 32), (8, 40)]:
    A = np.zeros((n, m), np.float32); A[:, bk] = np.arange(n)
    B = np.zeros((m, l), np.float32); B[bk, bj] = 1
    C = jb.matmul(A, B)
    nz = np.argwhere(C != 0)
    print(f" probe B[{bk},{bj}]=1, A[:,{bk}]=0..127 -> nonzero C cols {sorted(set(nz[:,1].tolist()))[:8]} rows {sorted(set(nz[:,0].tolist()))[:5]}")
# k-blocks: m=64 (two k-blocks)
n, m, l = 128, 64, 64
A = t(rng.integers(-3, 4, (n, m))); B = t(rng.integers(-3, 4, (m, l)))
C = jb.matmul(A, B); R = A @ B
print("2 kblocks int exact?", np.array_equal(C, R), np.abs(C - R).max())
n, m, l = 256, 256, 128
A = t(rng.integers(-3, 4, (n, m))); B = t(rng.integers(-3, 4, (m, l)))
C = jb.matmul(A, B); R = A @ B
print("256x256x128 int exact?", np.array_equal(C, R), np.abs(C - R).max())
A = rng.standard_normal((n, m)).astype(np.float32); B = rng.standard_normal((m, l)).astype(np.float32)
C = jb.matmul(A, B); R = (A.astype(np.float64) @ B.astype(np.float64))
print("256x256x128 float rel err", np.abs(C - R).max() / np.abs(R).max())
