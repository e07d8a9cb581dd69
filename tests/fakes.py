"""Numpy test doubles for the device layer (CPU tests only).

`NumpySpace` implements the DeviceLbfgs vector-space protocol with numpy
arrays and the oracle's split objective, so the device L-BFGS control flow
(dot-product two-loop, pair filter, precision switch) is testable without a
GPU.  `NumpyShardProblem` implements the DeviceProblem methods ShardedSpace
uses for one column shard, from the oracle's arithmetic.
"""

import numpy as np

from oracle import spcp_oracle as orc


class NumpySpace:
    def __init__(self, x, lam_l, lam_s, m, n, k, mask=None):
        self.x, self.lam_l, self.lam_s, self.mask = x, lam_l, lam_s, mask
        self.m, self.n, self.k = m, n, k
        self.length = (m + n) * k
        self.evals = 0

    def empty(self):
        return np.empty(self.length)

    def eval(self, z, d, alpha, g_out, precision):
        w = z if d is None else z + alpha * d
        f, g = orc.flat_objective(self.x, self.lam_l, self.lam_s, self.mask, self.m, self.n,
                                  self.k)(w)
        g_out[:] = g
        self.evals += 1
        gd = float(g @ d) if d is not None else 0.0
        return f, gd, float(g @ g)

    def gram(self, a_list, b_list):
        return np.array([[float(a @ b) for b in b_list] for a in a_list])

    def lincomb(self, coefs, vecs, out):
        acc = np.zeros_like(out)
        for c, v in zip(coefs, vecs):
            acc += c * v
        out[:] = acc
        return out

    def to_host(self, z):
        return np.asarray(z)


class NumpyShardProblem:
    """One column shard: the partial/finish split of spcp_eval_partial/_finish."""

    def __init__(self, x_local, lam_l, lam_s, torch_device="cpu"):
        import torch

        self.x = x_local
        self.m, self.n = x_local.shape
        self.lam_l, self.lam_s = lam_l, lam_s
        self.device = torch.device(torch_device)

    def empty(self, n):
        import torch

        return torch.empty(int(n), dtype=torch.float64)

    def _split(self, z, k):
        mk = self.m * k
        return z[:mk].reshape(self.m, k), z[mk:].reshape(self.n, k)

    def eval_partial(self, k, dtype, z, d, alpha, gu_part, scal, g_out):
        w = z.numpy() if d is None else z.numpy() + alpha * d.numpy()
        u, v = self._split(w, k)
        phi, gv_raw, gtu = orc.split_raw_products(u, v, self.x, self.lam_s)
        mk = self.m * k
        gvv = gtu + self.lam_l * v
        g_out[mk:] = __import__("torch").from_numpy(gvv.ravel())
        dv = d.numpy()[mk:] if d is not None else np.zeros(self.n * k)
        gu_part[:] = __import__("torch").from_numpy(gv_raw.ravel()).to(gu_part.dtype)
        scal[:] = __import__("torch").tensor([phi, 0.5 * self.lam_l * float(np.sum(v * v)),
                                              float(gvv.ravel() @ dv),
                                              float(gvv.ravel() @ gvv.ravel())],
                                             dtype=scal.dtype)

    def eval_finish(self, k, dtype, z, d, alpha, gu_sum, scal_sum, g_out):
        w = z.numpy() if d is None else z.numpy() + alpha * d.numpy()
        mk = self.m * k
        u = w[:mk]
        gu = gu_sum.double().numpy() + self.lam_l * u
        g_out[:mk] = __import__("torch").from_numpy(gu)
        du = d.numpy()[:mk] if d is not None else np.zeros(mk)
        s = scal_sum.numpy()
        reg_u = 0.5 * self.lam_l * float(u @ u)
        f = s[0] + reg_u + s[1]
        return np.array([f, s[0], reg_u + s[1], float(gu @ du) + s[2], float(gu @ gu) + s[3],
                         float(gu @ gu), float(gu @ du), 0.0])

    def vec_gram(self, a_list, b_list):
        return np.array([[float(a.double() @ b.double()) for b in b_list] for a in a_list])

    def lincomb(self, coefs, vecs, out):
        acc = vecs[0] * coefs[0]
        for c, v in zip(coefs[1:], vecs[1:]):
            acc = acc + c * v
        out.copy_(acc)
        return out


class NumpyCertProblem(NumpyShardProblem):
    """The DeviceProblem surface the certificate uses (gram, matmul_small,
    apply, f_zero) for one column shard, from the oracle's arithmetic on CPU
    torch tensors: certificate_core / certificate_sharded run unchanged."""

    def __init__(self, x_local, lam_l, lam_s, mask_local=None):
        super().__init__(x_local, lam_l, lam_s)
        self.mask = mask_local
        self.lambda_l = lam_l
        xo = x_local if mask_local is None else np.where(mask_local, x_local, 0.0)
        self.f_zero = 0.5 * float(np.sum(xo * xo))
        self.store = frozenset({"f64"})
        self.apply_calls = 0

    def gram(self, a, b):
        return a.double().numpy().T @ b.double().numpy()

    def matmul_small(self, a, mat):
        import torch

        return torch.from_numpy(a.double().numpy() @ np.asarray(mat, np.float64))

    def apply(self, k, z, w_right=None, w_left=None, precision="fp64"):
        import torch

        zz = z.numpy()
        u, v = self._split(zz, k)
        _, g, _ = orc.phi_value_grad(u @ v.T, self.x, self.lam_s, self.mask)
        self.apply_calls += 1
        left = torch.from_numpy(g @ w_right.numpy()) if w_right is not None else None
        right = torch.from_numpy(g.T @ w_left.numpy()) if w_left is not None else None
        return left, right
