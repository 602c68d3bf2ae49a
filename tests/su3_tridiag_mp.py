"""Test-side construction of the GPU's general spin-one Lie–Trotter factor (reading R20, GPU form) in
40-digit arithmetic — NOT part of the oracle.

The CUDA kernel exponentiates a general su(3) H through the unitary similarity W that makes S = W†HW real symmetric
tridiagonal (the Lanczos process started at the m = +1 basis vector), T₀ = e^{−iD/2n} e^{−iX/n} e^{−iD/2n} on
S = D + X (the paper's factor shape, Eq. lie_trotter_4), T = W T₀ W†, U = T^n.  The oracle instead follows
the paper's printed basis product in leapfrog order; the two are different second-order splittings and
agree only once τ is large (≥ 20).  Low-τ GPU results are therefore checked against THIS construction: W from an
mpmath Lanczos process (independent of the kernel's explicit Givens-plus-phase W), each factor by mpmath.expm, and the
n = 2^τ power by exact repeated squaring at 40 digits."""
import math

import mpmath
import numpy as np

R2 = 1 / math.sqrt(2)
JX = R2 * np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], complex)
JY = R2 * np.array([[0, -1j, 0], [1j, 0, -1j], [0, 1j, 0]], complex)
JZ = np.diag([1.0, 0.0, -1.0]).astype(complex)
Q = np.diag([1.0, -2.0, 1.0]).astype(complex) / 3
BASIS = [JX, JY, JZ, Q, JX @ JX - JY @ JY, JX @ JY + JY @ JX, JX @ JZ + JZ @ JX, JY @ JZ + JZ @ JY]


def H8(a):
    return sum(x * A for x, A in zip(a, BASIS))


def lanczos(Hm):
    """W = [q0, q1, q2] with W†HW real tridiagonal and positive off-diagonals, from q0 = e_{m=+1}."""
    q0 = mpmath.matrix([1, 0, 0])
    dot = lambda u, v: sum(mpmath.conj(u[i]) * v[i] for i in range(3))
    w = Hm * q0
    w = w - dot(q0, w) * q0
    b1 = mpmath.sqrt(mpmath.re(dot(w, w)))
    q1 = w / b1
    w = Hm * q1
    w = w - dot(q0, w) * q0 - dot(q1, w) * q1
    q2 = w / mpmath.sqrt(mpmath.re(dot(w, w)))
    return mpmath.matrix([[q[i] for q in (q0, q1, q2)] for i in range(3)])


def tridiag_factor(a, tau, dps=40):
    """(T − I, U = T^(2^τ)) of the GPU's factor for coefficients a[8] (generic couplings: H01, H12 ≠ 0)."""
    n = 2 ** tau
    Hf = H8(a)
    with mpmath.workdps(dps):
        Hm = mpmath.matrix([[mpmath.mpc(complex(Hf[i, j])) for j in range(3)] for i in range(3)])
        Wm = lanczos(Hm)
        S = Wm.H * Hm * Wm
        D = mpmath.diag([mpmath.re(S[i, i]) for i in range(3)])
        X = mpmath.matrix(3, 3)
        X[0, 1] = X[1, 0] = mpmath.re(S[0, 1])
        X[1, 2] = X[2, 1] = mpmath.re(S[1, 2])
        ex = lambda M, s: mpmath.expm(M * (-1j) * s / n)
        T = Wm * ex(D, mpmath.mpf(1) / 2) * ex(X, 1) * ex(D, mpmath.mpf(1) / 2) * Wm.H
        U = T
        for _ in range(tau):
            U = U * U
        res = T - mpmath.eye(3)
        return (np.array([[complex(res[i, j]) for j in range(3)] for i in range(3)]),
                np.array([[complex(U[i, j]) for j in range(3)] for i in range(3)]))
