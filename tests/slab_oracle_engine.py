"""The CPU oracle behind the slab runner's engine interface (test
infrastructure: lets the x-slab decomposition run on CPU ranks with gloo)."""
import contextlib

import numpy as np
import torch


class OracleEngine:
    device = "cpu"

    def __init__(self, oracle, cfg):
        self.o = oracle
        self.n, self.nb = oracle.n, oracle.nb
        self.iters, self.substeps = cfg.solver_iterations, cfg.substeps

    def context(self):
        return contextlib.nullcontext()

    def index(self, a):
        return torch.as_tensor(np.ascontiguousarray(a, np.int32))

    def gather(self, fld, idx):
        return torch.from_numpy(self.o.gather(fld, idx.numpy()))

    def scatter(self, fld, idx, values):
        self.o.scatter(fld, idx.numpy(), values.numpy())

    def set_roles(self, roles):
        self.o.set_roles(roles)

    def begin(self):
        self.o.integrate()
        self.o.candidates()

    def iteration(self):
        self.o.iteration()

    def end_substep(self):
        self.o.end_substep()

    def sync(self):
        st, bits, body, _ = self.o.error()
        if st != 0:
            raise RuntimeError(f"oracle error status {st} bits {bits} body {body}")

    def com_x(self):
        return self.o.body_stats()[:, 0]
