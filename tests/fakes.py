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


class NumpyLineSpace(NumpySpace):
    """NumpySpace with the stored-ray probes of spcp_line_setup / _probe
    (R(a) = R0 - a D1 - a^2 D2 on Omega), numpy float64."""

    def __init__(self, *a, fits=True, **kw):
        super().__init__(*a, **kw)
        self.fits = fits
        self.setups = self.releases = self.line_probes = 0
        self.ray = None

    def _uv(self, w):
        mk = self.m * self.k
        return w[:mk].reshape(self.m, self.k), w[mk:].reshape(self.n, self.k)

    def line_setup(self, z, d):
        self.setups += 1
        if not self.fits:
            return False
        u, v = self._uv(z)
        du, dv = self._uv(d)
        obs = np.ones_like(self.x, bool) if self.mask is None else self.mask.astype(bool)
        r0 = np.where(obs, self.x - u @ v.T, 0.0)
        d1 = np.where(obs, du @ v.T + u @ dv.T, 0.0)
        d2 = np.where(obs, du @ dv.T, 0.0)
        self.ray = (r0, d1, d2, float(z @ z), float(z @ d), float(d @ d))
        return True

    def line_probe(self, alpha):
        r0, d1, d2, zz, zd, dd = self.ray
        r = r0 - alpha * (d1 + alpha * d2)
        c = np.clip(r, -self.lam_s, self.lam_s)
        phi = float(np.sum(np.abs(c) * (np.abs(r) - 0.5 * np.abs(c))))
        dphi = float(np.sum(-c * (d1 + 2.0 * alpha * d2)))
        reg = 0.5 * self.lam_l * (zz + alpha * (2.0 * zd + alpha * dd))
        dreg = self.lam_l * (zd + alpha * dd)
        self.line_probes += 1
        return phi + reg, dphi + dreg

    def line_release(self):
        self.releases += 1
        self.ray = None


class NumpyLineShardProblem(NumpyShardProblem):
    """NumpyShardProblem with the stored-ray probes (spcp_line_*) of one shard:
    out = [F_p, phi_p, reg_p, gd_p, 0...] where reg_p covers [U | V_p]."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.lambda_l = self.lam_l
        self.ray = None
        self.setups = self.releases = 0

    def line_setup(self, k, z, d):
        zz, dd = z.double().numpy(), d.double().numpy()
        u, v = self._split(zz, k)
        du, dv = self._split(dd, k)
        self.ray = (self.x - u @ v.T, du @ v.T + u @ dv.T, du @ dv.T,
                    float(zz @ zz), float(zz @ dd), float(dd @ dd))
        self.setups += 1
        return True

    def line_probe(self, alpha):
        r0, d1, d2, zz, zd, dd = self.ray
        r = r0 - alpha * (d1 + alpha * d2)
        c = np.clip(r, -self.lam_s, self.lam_s)
        phi = float(np.sum(np.abs(c) * (np.abs(r) - 0.5 * np.abs(c))))
        dphi = float(np.sum(-c * (d1 + 2.0 * alpha * d2)))
        reg = 0.5 * self.lam_l * (zz + alpha * (2.0 * zd + alpha * dd))
        dreg = self.lam_l * (zd + alpha * dd)
        return np.array([phi + reg, phi, reg, dphi + dreg, 0.0, 0.0, 0.0, 0.0])

    def line_release(self):
        self.releases += 1
        self.ray = None
