"""ORACLE / TEST INFRASTRUCTURE ONLY.

A CPU engine with the slab-mode interface of paper_1507_06565_b200.Simulation
(step_part / step_finish / halo_parity / set_halo_buffers / get_pdfs / ...)
so the product's multi-rank stepping and halo exchange (dist.py) can be run
world_size > 1 over gloo on CPU and compared bit-for-bit with the
single-domain oracle.  It restates the pull form of the reference step
(SURVEY §8a-P): f_j(x) = g_j(x - e_j) with ghost columns for x - e_j outside
the slab, link closure (boundary.cpp:19-41 in pull form) and the reference
collision (oracle/porolb_oracle.c, orc_collide_core / orc_collide_glbm).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from oracle.oracle import OracleLib, _p, _v3

E = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1],
              [1, 1, 0], [-1, -1, 0], [1, -1, 0], [-1, 1, 0], [1, 0, 1], [-1, 0, -1], [1, 0, -1],
              [-1, 0, 1], [0, 1, 1], [0, -1, -1], [0, 1, -1], [0, -1, 1]])
OPP = np.array([0] + [k + 1 if k % 2 else k - 1 for k in range(1, 19)])
W = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
TO_RIGHT = (1, 7, 9, 11, 13)
TO_LEFT = (2, 8, 10, 12, 14)


class OracleSlabSim:
    def __init__(self, geom, workload):
        self.o = OracleLib()
        self.dims = tuple(geom.dims)
        nx, ny, nz = self.dims
        self.cells = nx * ny * nz
        self.flags = np.ascontiguousarray(geom.flags, dtype=np.uint8)
        self.fluid = self.flags.reshape(nz, ny, nx) == 0
        self.per = geom.periodic
        p = workload.params()
        self.wp, self.wm, self.rho0, self.nu = p.omega_plus, p.omega_minus, p.rho0, p.nu
        self.g = np.array(p.body_force, dtype=np.float64)
        self.scheme = int(workload.scheme)
        gp = workload.glbm_params()
        self.glbm = None if gp is None else tuple(np.ascontiguousarray(a, dtype=np.float64) for a in (
            gp.eps, gp.permeability, gp.omega_plus, gp.omega_minus))
        self.lf = np.asarray(geom.link_fluid_cell, dtype=np.int64)
        self.ld = np.asarray(geom.link_direction)
        self.ls = np.asarray(geom.link_second_fluid)
        self.lq = np.asarray(geom.link_q, dtype=np.float32).astype(np.float64)
        self.lm = np.asarray(geom.link_moving).astype(bool)
        self.fluid_cells = int(geom.fluid_cells)
        self.porosity = np.asarray(geom.porosity)
        self.state = np.zeros((19, nz, ny, nx))
        self.post = False
        self.pending = 0
        self.ghost_cur = 0
        self.steps_done = 0
        self.halo_elems = 5 * ny * nz
        self._next = None

    def set_halo_buffers(self, send_lo, send_hi, rl0, rl1, rh0, rh1):
        self.send_lo, self.send_hi = send_lo.numpy(), send_hi.numpy()
        self.recv_lo = [rl0.numpy(), rl1.numpy()]
        self.recv_hi = [rh0.numpy(), rh1.numpy()]

    @property
    def halo_parity(self):
        return 1 - self.ghost_cur

    # -- the pull step -------------------------------------------------------
    def _pull(self, g):
        nx, ny, nz = self.dims
        gl = self.recv_lo[self.ghost_cur].reshape(5, nz, ny)
        gh = self.recv_hi[self.ghost_cur].reshape(5, nz, ny)
        ext = np.zeros((19, nz, ny, nx + 2))
        ext[:, :, :, 1:-1] = g
        for s, j in enumerate(TO_RIGHT):
            ext[j, :, :, 0] = gl[s]
        for s, j in enumerate(TO_LEFT):
            ext[j, :, :, -1] = gh[s]
        F = np.empty_like(g)
        for j in range(19):
            ex, ey, ez = E[j]
            a = np.roll(ext[j], shift=(ez, ey), axis=(0, 1))  # value at (z - ez, y - ey)
            F[j] = a[:, :, 1 - ex:1 - ex + nx]
        # link closure in pull form
        Ff = F.reshape(19, -1)
        gf = g.reshape(19, -1)
        k = self.ld
        j = OPP[k]
        gk = gf[k, self.lf]
        val = gk.copy()
        cli = (~self.lm) & (self.scheme == 1) & (self.ls != -1)
        if cli.any():
            q = self.lq[cli]
            c = (1.0 - 2.0 * q) / (1.0 + 2.0 * q)
            A = Ff[k[cli], self.lf[cli]]  # pull value of direction k == g_k(x - e_k)
            B = gf[j[cli], self.lf[cli]]
            val[cli] = (c * A - c * B) + gk[cli]
        Ff[j, self.lf] = val
        return F

    def _collide(self, F):
        L = self.o.lib
        F = np.ascontiguousarray(F)
        if self.glbm is not None:
            e, K, wp, wm = self.glbm
            L.orc_collide_glbm(self.cells, self.dims[0] * self.dims[1], _p(self.flags, C.c_uint8),
                               _p(F, C.c_double), self.rho0, self.nu, _v3(self.g), _p(e, C.c_double),
                               _p(K, C.c_double), _p(wp, C.c_double), _p(wm, C.c_double), 0.0, 1)
        else:
            L.orc_collide_core(self.cells, _p(self.flags, C.c_uint8), _p(F, C.c_double), self.wp,
                               self.wm, self.rho0, _v3(self.g))
        return F

    def _send(self, g):
        nx, ny, nz = self.dims
        for s, j in enumerate(TO_LEFT):
            self.send_lo.reshape(5, nz, ny)[s] = g[j, :, :, 0]
        for s, j in enumerate(TO_RIGHT):
            self.send_hi.reshape(5, nz, ny)[s] = g[j, :, :, nx - 1]

    def step_part(self, part):
        if part == 0:
            if not self.post:
                self._next = self._collide(self.state.copy())
                self.pending = 1
            else:
                F = self._pull(self.state)
                self._next = self._collide(F)
                self.pending = 2
            self._next[:, ~self.fluid] = 0.0
            self._send(self._next)

    def step_finish(self):
        self.state = self._next
        self.post = True
        self.pending = 0
        self.ghost_cur = 1 - self.ghost_cur
        self.steps_done += 1

    def get_pdfs(self):
        if not self.post:
            return self.state.copy()
        F = self._pull(self.state)
        F[:, ~self.fluid] = 0.0
        return F

    # -- observables used by dist.DistTransport (tolerance-level, test only) --
    def _macro(self):
        f = self.get_pdfs()
        d = np.zeros(f.shape[1:])
        u = [np.zeros(f.shape[1:]) for _ in range(3)]
        for k in range(19):  # lattice.cpp:88-101 order
            d = d + f[k]
            for i in range(3):
                u[i] = u[i] + E[k][i] * f[k]
        u = [ui / self.rho0 + 0.5 * self.g[i] / self.rho0 for i, ui in enumerate(u)]
        return d, u

    def plane_sums(self, axis=0):
        _, u = self._macro()
        return np.where(self.fluid, u[axis], 0.0).sum(axis=(1, 2))

    def max_speed2(self):
        d, u = self._macro()
        m2 = (u[0] * u[0] + u[1] * u[1]) + u[2] * u[2]
        m2 = np.where(self.fluid, m2, 0.0)
        fin = bool(np.all(np.isfinite(m2)) and np.all(np.isfinite(np.where(self.fluid, d, 0.0))))
        return float(np.nanmax(m2)), fin
