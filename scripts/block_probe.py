import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1911_01492_b200 as pb
A = pb.q1_device((128,)*3)
S = pb.spai1_symmetric_device(A)
B = pb.MultiVector(np.random.default_rng(0).standard_normal((A.nrows, 4)))
X, recs = pb.block_solve(A, B, pb.SparseMatrixPreconditioner(S), pb.SolverConfig(tol=1e-8, maxit=60), gram_mode="full")
print(max(r.iterations for r in recs))
