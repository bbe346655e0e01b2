"""Small dense/CSR helpers shared by the tests (no method arithmetic)."""
import numpy as np


def csr_from_dense_diaglast(A):
    n = A.shape[0]
    rowptr = [0]; col = []; val = []
    for i in range(n):
        nz = [j for j in range(n) if j != i and A[i, j] != 0]
        col += nz + [i]; val += [A[i, j] for j in nz] + [A[i, i]]
        rowptr.append(len(col))
    return np.array(rowptr, np.int64), np.array(col, np.int32), np.array(val, float)


def dense(rowptr, col, val, n=None):
    n = n or rowptr.shape[0] - 1
    A = np.zeros((rowptr.shape[0] - 1, n))
    for i in range(rowptr.shape[0] - 1):
        A[i, col[rowptr[i]:rowptr[i + 1]]] = val[rowptr[i]:rowptr[i + 1]]
    return A
