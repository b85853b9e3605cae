"""TEST INFRASTRUCTURE: a numpy/torch-CPU implementation of the local compute
steps of paper_1903_07884_b200.dist, so the sharded solve's data movement
(layouts, pack/unpack, all-to-all splits, all-reduces, GMRES control) can be
exercised on CPU with the gloo backend.  Local arithmetic follows the oracle
(oracle/voxvie_oracle.py)."""

import numpy as np
import scipy.fft
import torch
from scipy.linalg import lu_factor, lu_solve

import voxvie_oracle as O

PAIR_OF = O.PAIR_OF


class NumpyBackend:
    def empty(self, shape):
        return torch.zeros(shape, dtype=torch.complex128)

    def ints(self, a):
        return torch.from_numpy(np.ascontiguousarray(a, np.int64))

    def to_dev(self, a):
        return torch.from_numpy(np.ascontiguousarray(a, np.complex128))

    def spectra(self, kernel):
        return torch.from_numpy(O.plan_spectra(kernel.tensors, kernel.grid.dims))

    def x_forward(self, x_loc, nl, nx, px):
        return torch.from_numpy(scipy.fft.fft(x_loc.numpy().reshape(nl, nx), px, axis=1))

    def op_yz(self, A, spectra_loc, dims, nkx, px, py, pz):
        nx, ny, nz = dims
        a = A.numpy().reshape(3, nz, ny, nkx)
        ah = scipy.fft.fft(scipy.fft.fft(a, py, axis=2), pz, axis=1)
        s = spectra_loc.numpy()
        out = np.empty_like(a)
        for p in range(3):
            acc = s[PAIR_OF[p, 0]] * ah[0] + s[PAIR_OF[p, 1]] * ah[1] + s[PAIR_OF[p, 2]] * ah[2]
            out[p] = scipy.fft.ifft(scipy.fft.ifft(acc, axis=1), axis=0)[:nz, :ny]
        A.copy_(torch.from_numpy(out.reshape(-1)))

    def x_inverse(self, A, dims, px, nl, line0, m_full, x_loc):
        nx, ny, nz = dims
        v = scipy.fft.ifft(A.numpy().reshape(nl, px), axis=1)[:, :nx].reshape(-1)
        if m_full is not None:
            m = m_full.numpy().reshape(-1)
            idx = (line0 * nx + np.arange(nl * nx)) % (nx * ny * nz)
            v = x_loc.numpy() - m[idx] * v
        return torch.from_numpy(np.ascontiguousarray(v))

    def dft_lines(self, x, nl, n, inverse):
        a = x.numpy().reshape(nl, n)
        return torch.from_numpy((scipy.fft.ifft if inverse else scipy.fft.fft)(a, axis=1))

    def gather_cols(self, A, nrows, lda, col_off, colmap, total):
        a = A.numpy().reshape(nrows, lda)
        off, cm = col_off.numpy(), colmap.numpy()
        parts = [a[:, cm[off[s]:off[s + 1]]].reshape(-1) for s in range(len(off) - 1)]
        return torch.from_numpy(np.concatenate(parts + [np.zeros(1, complex)]))

    def scatter_cols(self, buf, A, nrows, lda, col_off, colmap, total):
        a = A.numpy().reshape(nrows, lda)
        off, cm = col_off.numpy(), colmap.numpy()
        b = buf.numpy()
        pos = 0
        for s in range(len(off) - 1):
            nc = off[s + 1] - off[s]
            a[:, cm[off[s]:off[s + 1]]] = b[pos:pos + nrows * nc].reshape(nrows, nc)
            pos += nrows * nc

    def chan_x(self, kernel):
        return O.chan_x_spectra(kernel.tensors)

    def proxies(self, lam, dims, m00):
        nx, ny, nz = dims
        return (1.0 if ny * nz == 1 else 0.0) - m00 * lam[0, 0, 0, :]

    def build_factors(self, lam, dims, m_yz, kset):
        facs = [O.lu_checked(O.unfold_block_yz(lam[:, :, :, int(k)], m_yz)) for k in kset]
        return facs, None

    def chan_xy(self, kernel):
        # (6, 2nz-1, ny, nx): Chan along x then y, 2-D DFT (oracle build_two_level)
        return scipy.fft.fftn(O.chan_along_axis(O.chan_along_axis(kernel.tensors, 3), 2), axes=(2, 3))

    def build_factors2(self, lam2, dims, m_z, kset):
        nx, ny, nz = dims
        facs = []
        for key in kset:
            l, k = divmod(int(key), nx)
            facs.append(O.lu_checked(O.unfold_block_z(lam2[:, :, l, k], m_z)))
        return facs, None

    def dft_y(self, Y, nplanes, ny, nk, inverse):
        a = Y.numpy()[: nplanes * ny * nk].reshape(nplanes, ny, nk)
        a[...] = (scipy.fft.ifft if inverse else scipy.fft.fft)(a, axis=1)

    def solve(self, Y, n, factors, perm, items, n_single, n_items, klist, s_row):
        y = Y.numpy()[: n * s_row].reshape(n, s_row)
        it = items.numpy().reshape(-1, 3)
        kl = klist.numpy()
        for slot, beg, cnt in it[:n_items]:
            for c in kl[beg:beg + cnt]:
                y[:, c] = lu_solve(factors[slot], y[:, c], check_finite=False)

    def part(self, n, nvec):
        return None

    def cgs_dots(self, V, nvec, w, part):
        v = V.numpy()
        wn = w.numpy()
        out = np.empty(nvec + 1, complex)
        for i in range(nvec):
            out[i] = np.vdot(v[i], wn)
        out[nvec] = np.vdot(wn, wn).real
        return torch.from_numpy(out)

    def cgs_update(self, V, nvec, coef, w, part):
        v = V.numpy()
        c = coef.numpy()
        wn = w.numpy()
        for i in range(nvec):
            wn -= c[i] * v[i]
        return torch.from_numpy(np.array([np.vdot(wn, wn).real + 0j]))

    def axpby(self, a, x, b, y, out=None):
        r = complex(a) * x + (complex(b) * y if y is not None else 0)
        if out is None:
            return r.clone() if isinstance(r, torch.Tensor) else r
        out.copy_(r)
        return out

    def combine(self, V, nvec, y):
        return torch.from_numpy(np.asarray(y) @ V.numpy()[:nvec])

    def combine_list(self, zs, y):
        return torch.from_numpy(sum(complex(c) * z.numpy() for c, z in zip(np.asarray(y), zs)))

    def to_host(self, t):
        return t.numpy()
