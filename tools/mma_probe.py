import ctypes, numpy as np, os, subprocess, sys
here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "mma_probe.so")
lib = ctypes.CDLL(so)
rng = np.random.default_rng(0)
A = rng.integers(-3, 4, (128, 32)).astype(np.float32)
B = rng.integers(-3, 4, (32, 64)).astype(np.float32)
P = ctypes.POINTER(ctypes.c_float)
for mode in [1, 3, 8, 10, 12, 14]:
    C = np.zeros((128, 64), np.float32); dbg = np.zeros(6, np.float32)
    rc = lib.run_probe(A.ctypes.data_as(P), B.ctypes.data_as(P), C.ctypes.data_as(P), dbg.ctypes.data_as(P), mode)
    K = 32 if mode & 2 else 8
    R = A[:, :K] @ B[:K]
    print(f"mode {mode} (B {'K' if mode&1 else 'MN'}-major, K={K}) rc={rc} exact={np.array_equal(C, R)} maxerr={np.abs(C-R).max()} C00={C[0,:4]} R00={R[0,:4]} dbg={[hex(x) for x in dbg.view(np.uint32)]}")

# truncation probe: A has low mantissa bits set, B = identity block (K-major)
A = (rng.standard_normal((128, 32))).astype(np.float32)
B = np.zeros((32, 64), np.float32); B[np.arange(32), np.arange(32)] = 1
C = np.zeros((128, 64), np.float32); dbg = np.zeros(6, np.float32)
lib.run_probe(A.ctypes.data_as(P), B.ctypes.data_as(P), C.ctypes.data_as(P), dbg.ctypes.data_as(P), 3)
u = A.view(np.uint32)
trunc = (u & 0xFFFFE000).view(np.float32)
rnd = ((u + 0x1000) & 0xFFFFE000).view(np.float32)
got = C[:, :32]
print("tf32 operand semantics: equals truncation:", np.array_equal(got, trunc), " equals rna:", np.array_equal(got, rnd),
      " equals fp32:", np.array_equal(got, A), " max|got-A|/|A|", np.max(np.abs(got - A) / np.abs(A)))
