"""Run outputs: dense macroscopic fields, legacy
VTK and CSV writers, and the convergence estimator.

Fields come off the device once (the solver's readout kernel + a device
scatter to the dense grid); the writers are host formatting only and are
deterministic (same inputs -> byte-identical files, SPEC acceptance 12).
"""

import numpy as np
import torch


def dense_macroscopic(solver):
    """(rho, u) on the dense (nx, ny, nz) grid as numpy; 0 at solid nodes."""
    rho, u, _ = solver.macroscopic(device=True)
    mask = solver.to_dense((solver.tiling.meta & 1).to(rho.dtype))
    r = solver.to_dense(rho) * mask
    v = solver.to_dense(u) * mask
    return r.cpu().numpy(), v.cpu().numpy()


def write_vtk(path_or_stream, rho, u, title="tiled D3Q19 LBM output"):
    """Legacy ASCII STRUCTURED_POINTS: density scalars + velocity vectors, x
    fastest (VTK point order)."""
    nx, ny, nz = rho.shape
    lines = ["# vtk DataFile Version 3.0", title[:255], "ASCII",
             "DATASET STRUCTURED_POINTS", f"DIMENSIONS {nx} {ny} {nz}", "ORIGIN 0 0 0",
             "SPACING 1 1 1", f"POINT_DATA {nx * ny * nz}",
             "SCALARS density double 1", "LOOKUP_TABLE default"]
    r = np.asarray(rho, dtype=np.float64).transpose(2, 1, 0).ravel()
    lines += [f"{v:.17g}" for v in r]
    lines.append("VECTORS velocity double")
    v = np.asarray(u, dtype=np.float64).transpose(3, 2, 1, 0).reshape(-1, 3)
    lines += [f"{a:.17g} {b:.17g} {c:.17g}" for a, b, c in v]
    text = "\n".join(lines) + "\n"
    if hasattr(path_or_stream, "write"):
        path_or_stream.write(text)
    else:
        with open(path_or_stream, "w") as fh:
            fh.write(text)


def write_csv_slice(path, rho, u, axis=2, index=None):
    """One axis-normal plane: columns x, y, z, rho, ux, uy, uz."""
    nx, ny, nz = rho.shape
    index = (rho.shape[axis] // 2) if index is None else int(index)
    sl = [slice(None)] * 3
    sl[axis] = index
    grid = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"))
    cols = [grid[a][tuple(sl)].ravel() for a in range(3)]
    cols.append(rho[tuple(sl)].ravel())
    cols += [u[a][tuple(sl)].ravel() for a in range(3)]
    with open(path, "w") as fh:
        fh.write("x,y,z,rho,ux,uy,uz\n")
        for row in zip(*cols):
            fh.write("%d,%d,%d,%.17g,%.17g,%.17g,%.17g\n" % row)


class ConvergenceEstimator:
    """Relative L2 change of u between checks: every ``every``
    steps, ||u_t - u_prev|| / ||u_t|| over non-solid slots, on the device."""

    def __init__(self, solver, every):
        self.solver, self.every = solver, int(every)
        self.prev = None
        self.history = []

    def __call__(self):
        _, u, _ = self.solver.macroscopic(device=True)
        mask = self.solver.nonsolid_mask(device=True)
        cur = u[:, mask].double()
        if self.prev is not None:
            num = torch.linalg.vector_norm(cur - self.prev)
            den = torch.linalg.vector_norm(cur)
            self.history.append((self.solver.iteration,
                                 float(num / den) if float(den) > 0 else 0.0))
        self.prev = cur
        return self.history[-1][1] if self.history else None
