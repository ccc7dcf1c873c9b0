"""Voxel geometry: node tags, the benchmark generators and TLBM1 voxel I/O.

Same data model as ``tilelbm.geometry`` (reference ``geometry.py:17-342``): a
dense ``uint8`` grid ``types[x, y, z]`` in C order (z fastest in memory) plus a
uniform inlet velocity and outlet density.  Geometry generation is *input
preparation* for the hot path (it runs once per case, on the host, exactly as
in the reference); everything downstream of it -- tiling, metadata, the step,
readout -- runs on the GPU.

Extensions over the reference (all documented in DESIGN.md):

* ``Geometry.periodic`` -- per-axis periodic wrap of the pull gather.  The
  reference treats off-domain as SOLID; BASELINE config 2 needs
  a periodic channel, so the flag defaults to all-False (reference behaviour).
* ``generate_channel(..., ends="periodic")`` -- no end caps, periodic along the
  channel axis.
* ``generate_box`` -- the porosity-1.0 end of the sphere-pack sweep, which
  ``generate_sphere_pack`` rejects (geometry.py:218-219).
* ``generate_vessel_tree`` -- seeded bifurcating-tube geometry for config 4.
* ``device=`` on both generators builds the voxels on the GPU
  (csrc/generate.cu), bit-identical to the host path.
* ``generate_sphere_pack`` draws the identical random sequence as the
  reference but rasterises each sphere only inside its bounding box, so the
  result is bit-identical and O(d^3) per sphere instead of O(n^3).
"""

import enum
import json
from dataclasses import dataclass

import numpy as np


class NodeType(enum.IntEnum):
    SOLID = 0
    FLUID = 1
    BB_WALL = 2
    VELOCITY_INLET = 3
    PRESSURE_OUTLET = 4


VOXEL_MAGIC = b"TLBM1"
_TAGS = frozenset(int(t) for t in NodeType)


class VoxelFormatError(ValueError):
    """Malformed TLBM1 stream (geometry.py:30-31)."""


@dataclass
class Geometry:
    types: np.ndarray
    inlet_velocity: tuple = (0.0, 0.0, 0.0)
    outlet_density: float = 1.0
    periodic: tuple = (False, False, False)

    def __post_init__(self):
        self.types = np.ascontiguousarray(self.types, dtype=np.uint8)
        if self.types.ndim != 3:
            raise ValueError("types array must be 3-dimensional")
        vel = tuple(float(v) for v in self.inlet_velocity)
        if len(vel) != 3:
            raise ValueError("inlet velocity must be a 3-component vector")
        self.inlet_velocity = vel
        self.outlet_density = float(self.outlet_density)
        per = tuple(bool(p) for p in self.periodic)
        if len(per) != 3:
            raise ValueError("periodic must name 3 axes")
        for axis, p in enumerate(per):
            if p and self.types.shape[axis] % 4:
                raise ValueError(
                    f"periodic axis {axis} needs a multiple of 4 nodes, got "
                    f"{self.types.shape[axis]}")
        self.periodic = per

    @property
    def shape(self):
        return self.types.shape

    @property
    def node_count(self):
        return int(self.types.size)

    def nonsolid_mask(self):
        return self.types != NodeType.SOLID

    def nonsolid_count(self):
        return int(np.count_nonzero(self.types))

    def porosity(self):
        return self.nonsolid_count() / self.node_count

    def __eq__(self, other):
        if not isinstance(other, Geometry):
            return NotImplemented
        return (self.types.shape == other.types.shape
                and bool(np.array_equal(self.types, other.types))
                and self.inlet_velocity == other.inlet_velocity
                and self.outlet_density == other.outlet_density
                and self.periodic == other.periodic)


def _face_slice(axis, index):
    sl = [slice(None)] * 3
    sl[axis] = index
    return tuple(sl)


def generate_cavity3d(b, lid_velocity=(0.05, 0.0, 0.0)):
    """Lid-driven cube (geometry.py:80-99): BB walls on all six faces, the
    interior of the +z face a velocity inlet; wall rims win at edges."""
    b = int(b)
    if b < 4:
        raise ValueError(f"cavity edge must be at least 4 nodes, got {b}")
    t = np.full((b, b, b), NodeType.BB_WALL, dtype=np.uint8)
    t[1:-1, 1:-1, 1:-1] = NodeType.FLUID
    t[1:-1, 1:-1, b - 1] = NodeType.VELOCITY_INLET
    return Geometry(t, inlet_velocity=lid_velocity)


def _cross_section(shape, d, off1, off2):
    """(inside, interior) masks of one channel cross-section
    (geometry.py:102-133): square = d x d block; circle = cell centres strictly
    inside the disc of diameter d+1; interior = 4-neighbourhood inside."""
    n1, n2 = off1 + d, off2 + d
    a = np.arange(n1)[:, None]
    b = np.arange(n2)[None, :]
    if shape == "square":
        inside = ((a >= off1) & (a < off1 + d)) & ((b >= off2) & (b < off2 + d))
    elif shape == "circle":
        r1 = 2 * (a - off1) - (d - 1)
        r2 = 2 * (b - off2) - (d - 1)
        inside = r1 * r1 + r2 * r2 < (d + 1) ** 2
    else:
        raise ValueError(f"unknown channel shape: {shape!r}")
    p = np.pad(inside, 1, constant_values=False)
    interior = inside & p[:-2, 1:-1] & p[2:, 1:-1] & p[1:-1, :-2] & p[1:-1, 2:]
    return inside, interior


def generate_channel(shape, d, axis=0, offsets=(0, 0), length=16, ends="wall",
                     inlet_velocity=(0.0, 0.0, 0.0), outlet_density=1.0):
    """Straight square/circular channel in solid (geometry.py:136-197).

    ``ends``: "wall" (BB caps), "io" (inlet low end, outlet high end) or the
    extension "periodic" (no caps, periodic along ``axis``; ``length`` must be
    a multiple of 4).
    """
    d = int(d)
    if d < 1:
        raise ValueError(f"channel cross-section must be >= 1 node, got {d}")
    off1, off2 = (int(o) for o in offsets)
    if not (0 <= off1 <= 3 and 0 <= off2 <= 3):
        raise ValueError(f"offsets must be in 0..3, got {offsets}")
    length = int(length)
    if length < 1:
        raise ValueError(f"channel length must be >= 1, got {length}")
    axis = int(axis)
    if axis not in (0, 1, 2):
        raise ValueError(f"axis must be 0, 1 or 2, got {axis}")
    inside, interior = _cross_section(shape, d, off1, off2)
    if not inside.any():
        raise ValueError("channel cross-section is empty")
    cross = np.zeros(inside.shape, dtype=np.uint8)
    cross[inside] = NodeType.BB_WALL
    cross[interior] = NodeType.FLUID

    trans = [a for a in range(3) if a != axis]
    dims = [0, 0, 0]
    dims[axis] = length
    dims[trans[0]], dims[trans[1]] = cross.shape
    t = np.empty(dims, dtype=np.uint8)
    np.moveaxis(t, axis, 2)[...] = cross[:, :, None]

    periodic = [False, False, False]
    lo, hi = t[_face_slice(axis, 0)], t[_face_slice(axis, length - 1)]
    if ends == "wall":
        lo[lo != NodeType.SOLID] = NodeType.BB_WALL
        hi[hi != NodeType.SOLID] = NodeType.BB_WALL
    elif ends == "io":
        lo[lo == NodeType.FLUID] = NodeType.VELOCITY_INLET
        hi[hi == NodeType.FLUID] = NodeType.PRESSURE_OUTLET
    elif ends == "periodic":
        periodic[axis] = True
    else:
        raise ValueError(f"unknown ends mode: {ends!r}")
    return Geometry(t, inlet_velocity=inlet_velocity,
                    outlet_density=outlet_density, periodic=tuple(periodic))


def _sphere_pack_device(n, r, target, seed, max_passes, device):
    """Solid/fluid tags of the sphere pack, built on the GPU (see
    generate_sphere_pack).  Same RNG stream, same stopping rule:
    porosity(k) = 1 - solid(k) / n^3 with solid(k) the voxels whose first
    covering sphere is among the pass's first k; the pass stops at the
    smallest k with porosity(k) <= target + band and is accepted when
    porosity(k) >= target - band, else the next pass starts at sphere k."""
    import torch

    from . import _native as nat
    dev = nat.require_cuda(device)
    band = 0.005
    size = n * n * n
    rng = np.random.default_rng(seed)
    vol = 4.0 / 3.0 * np.pi * r ** 3
    batch = int(max(64, 1.3 * np.log(1.0 / max(target, 1e-3)) * size / max(vol, 1.0) + 64))
    drawn = np.empty((0, 3))
    start = 0                      # first sphere of the current pass
    big = np.iinfo(np.int32).max
    first = torch.full((n, n, n), big, dtype=torch.int32, device=dev)
    for _ in range(int(max_passes)):
        first.fill_(big)
        covered = start            # spheres of this pass already applied
        k_stop = None
        while k_stop is None:
            if drawn.shape[0] < covered + batch:
                drawn = np.concatenate([drawn, rng.uniform(0.0, n, size=(batch, 3))])
            c = torch.from_numpy(np.ascontiguousarray(drawn[covered:covered + batch])).to(dev)
            nat.call("tlbm_sphere_cover", nat.ptr(c), covered, batch, n, r, nat.ptr(first),
                     nat.stream_ptr(dev))
            covered += batch
            idx = first[first < covered] - start
            counts = torch.bincount(idx.to(torch.int64), minlength=covered - start)
            solid = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev),
                               torch.cumsum(counts, 0)]).cpu().numpy()
            porosity = 1.0 - solid / size
            hit = np.flatnonzero(porosity <= target + band)
            if hit.size:
                k_stop = int(hit[0])
        if porosity[k_stop] >= target - band:
            solid_mask = (first < start + k_stop).cpu().numpy()
            return np.where(solid_mask, np.uint8(NodeType.SOLID),
                            np.uint8(NodeType.FLUID)).astype(np.uint8)
        start += k_stop            # the next pass continues the RNG stream
    raise ValueError(f"target porosity {target} unreachable within +/-{band} after "
                     f"{max_passes} packing passes")


def _type_box_faces(t, flow_axis):
    """Inlet/outlet on the two flow-axis faces, BB on the other four, walls
    winning shared edges (geometry.py:251-266)."""
    n_lo = t[_face_slice(flow_axis, 0)]
    n_lo[n_lo == NodeType.FLUID] = NodeType.VELOCITY_INLET
    n_hi = t[_face_slice(flow_axis, t.shape[flow_axis] - 1)]
    n_hi[n_hi == NodeType.FLUID] = NodeType.PRESSURE_OUTLET
    for axis in range(3):
        if axis == flow_axis:
            continue
        for idx in (0, t.shape[axis] - 1):
            w = t[_face_slice(axis, idx)]
            w[w != NodeType.SOLID] = NodeType.BB_WALL


def generate_sphere_pack(n, diameter, target_porosity, seed, flow_axis=2,
                         inlet_velocity=(0.0, 0.0, 0.0), outlet_density=1.0,
                         max_passes=20, device=None):
    """Seeded overlapping solid spheres until porosity is within +/-0.005 of
    the target (geometry.py:200-269).

    Draws the same ``default_rng(seed).uniform(0, n, 3)`` centre sequence and
    applies the same ``(x+0.5-c)^2 sums <= r^2`` test as the reference, but
    only inside each sphere's bounding box, keeping a running solid count;
    the resulting voxels are bit-identical (tests/test_geometry.py).

    ``device`` (extension): build the pack on that CUDA device instead
    (csrc/generate.cu) -- every voxel records its first covering sphere and
    the stopping sphere follows from the per-sphere counts; same voxels.
    """
    n = int(n)
    if n < 4:
        raise ValueError(f"box edge must be at least 4 nodes, got {n}")
    if not 0.0 < target_porosity < 1.0:
        raise ValueError(f"target porosity must be in (0, 1): {target_porosity}")
    if device is not None:
        t = _sphere_pack_device(n, float(diameter) / 2.0, target_porosity, seed, max_passes,
                                device)
        _type_box_faces(t, flow_axis)
        return Geometry(t, inlet_velocity=inlet_velocity, outlet_density=outlet_density)
    r = float(diameter) / 2.0
    rr = r * r
    band = 0.005
    rng = np.random.default_rng(seed)
    centres = np.arange(n) + 0.5
    size = n * n * n

    for _ in range(int(max_passes)):
        solid = np.zeros((n, n, n), dtype=bool)
        count = 0
        while True:
            porosity = 1.0 - count / size
            if porosity <= target_porosity + band:
                break
            c = rng.uniform(0.0, n, size=3)
            d = [(centres - c[k]) ** 2 for k in range(3)]
            span = []
            for k in range(3):
                hit = np.flatnonzero(d[k] <= rr)
                span.append((int(hit[0]), int(hit[-1]) + 1) if hit.size else None)
            if any(s is None for s in span):
                continue
            (x0, x1), (y0, y1), (z0, z1) = span
            ball = (d[0][x0:x1, None, None] + d[1][None, y0:y1, None]
                    + d[2][None, None, z0:z1]) <= rr
            sub = solid[x0:x1, y0:y1, z0:z1]
            count += int(np.count_nonzero(ball & ~sub))
            sub |= ball
        if porosity >= target_porosity - band:
            break
    else:
        raise ValueError(
            f"target porosity {target_porosity} unreachable within "
            f"+/-{band} after {max_passes} packing passes")

    t = np.where(solid, np.uint8(NodeType.SOLID), np.uint8(NodeType.FLUID))
    t = t.astype(np.uint8)
    _type_box_faces(t, flow_axis)
    return Geometry(t, inlet_velocity=inlet_velocity,
                    outlet_density=outlet_density)


def generate_box(n, flow_axis=2, inlet_velocity=(0.0, 0.0, 0.0),
                 outlet_density=1.0):
    """Porosity-1.0 member of the sphere-pack family: the same face typing on
    an all-fluid box (SPEC.md:126 expects it; the reference generator rejects
    porosity >= 1)."""
    n = int(n)
    if n < 4:
        raise ValueError(f"box edge must be at least 4 nodes, got {n}")
    t = np.full((n, n, n), NodeType.FLUID, dtype=np.uint8)
    _type_box_faces(t, flow_axis)
    return Geometry(t, inlet_velocity=inlet_velocity,
                    outlet_density=outlet_density)


def generate_vessel_tree(shape=(512, 512, 1024), levels=3, root_radius=None,
                         seed=1234, wiggle=0.06, inlet_velocity=(0.0, 0.0, 0.01),
                         outlet_density=1.0, device=None):
    """Seeded tortuous bifurcating tube tree along +z (BASELINE config 4).

    A root tube enters at the centre of the z=0 face and bifurcates ``levels``
    times; every generation alternates the split plane (x, then y, ...),
    shrinks its radius by Murray's law (r / 2^(1/3)) and gets a seeded
    sinusoidal meander.  The leaves run to the z=nz-1 face.  Lumen nodes within
    a tube are non-solid; lumen nodes with a 6-neighbour outside the lumen are
    BB_WALL, the rest FLUID; fluid nodes on z=0 become VELOCITY_INLET and on
    z=nz-1 PRESSURE_OUTLET.  Tubes keep a margin from the x/y faces, so every
    inlet/outlet node lies on exactly one domain face.  Built slice by slice
    in O(nx*ny*nz) time.

    ``device`` (extension): rasterise and classify on that CUDA device
    (csrc/generate.cu) from the same per-slice branch discs; bit-identical
    voxels, a few hundred milliseconds instead of tens of seconds at
    1024x1024x2048.
    """
    nx, ny, nz = (int(v) for v in shape)
    rng = np.random.default_rng(seed)
    if root_radius is None:
        root_radius = 0.16 * min(nx, ny)
    seg = nz / (levels + 1)
    # tree[level] = [(dx, dy, r, parent index)]; a branch of level L is active
    # for z in [L*seg, (L+1)*seg)
    tree = {0: [(0.0, 0.0, float(root_radius), None)]}
    for lev in range(1, levels + 1):
        tree[lev] = []
        for pi, (px, py, pr, _) in enumerate(tree[lev - 1]):
            r = pr / 2.0 ** (1.0 / 3.0)
            spread = 1.15 * pr
            for s in (-1.0, 1.0):
                if lev % 2 == 1:
                    tree[lev].append((px + s * spread, py, r, pi))
                else:
                    tree[lev].append((px, py + s * spread, r, pi))
    phase = {lev: rng.uniform(0, 2 * np.pi, size=(len(tree[lev]), 2))
             for lev in tree}
    lam = {lev: rng.uniform(0.5, 1.0, size=len(tree[lev])) * seg for lev in tree}
    cx0, cy0 = (nx - 1) / 2.0, (ny - 1) / 2.0
    smooth = 0.35 * seg

    def centre(lev, i, z):
        px, py, r, parent = tree[lev][i]
        z0 = lev * seg
        if parent is not None:
            # blend from the parent's centre over the first part of the segment
            ppx, ppy, _, _ = tree[lev - 1][parent]
            w = min(1.0, max(0.0, (z - z0) / smooth))
            w = w * w * (3 - 2 * w)
            px = ppx + w * (px - ppx)
            py = ppy + w * (py - ppy)
        amp = wiggle * r * (1.0 if parent is not None else 0.5)
        ph = phase[lev][i]
        wx = amp * np.sin(2 * np.pi * z / lam[lev][i] + ph[0])
        wy = amp * np.sin(2 * np.pi * z / lam[lev][i] + ph[1])
        return cx0 + px + wx, cy0 + py + wy, r

    margin = 2.0
    if device is not None:
        t = _vessel_device(nx, ny, nz, [
            [centre(min(levels, int(z // seg)), i, float(z))
             for i in range(len(tree[min(levels, int(z // seg))]))] for z in range(nz)],
            int(margin), device)
        return Geometry(t, inlet_velocity=inlet_velocity, outlet_density=outlet_density)
    X = np.arange(nx, dtype=np.float64)[:, None]
    Y = np.arange(ny, dtype=np.float64)[None, :]
    lumen = np.zeros((nx, ny, nz), dtype=bool)
    for z in range(nz):
        lev = min(levels, int(z // seg))
        sl = lumen[:, :, z]
        for i in range(len(tree[lev])):
            cx, cy, r = centre(lev, i, float(z))
            x0, x1 = max(0, int(cx - r - 1)), min(nx, int(cx + r + 2))
            y0, y1 = max(0, int(cy - r - 1)), min(ny, int(cy + r + 2))
            dx = X[x0:x1] - cx
            dy = Y[:, y0:y1] - cy
            sl[x0:x1, y0:y1] |= dx * dx + dy * dy <= r * r
    lumen[:int(margin)] = False
    lumen[nx - int(margin):] = False
    lumen[:, :int(margin)] = False
    lumen[:, ny - int(margin):] = False
    p = np.pad(lumen, 1, constant_values=False)
    p[:, :, 0] = p[:, :, 1]          # the z faces are open (inlet/outlet)
    p[:, :, -1] = p[:, :, -2]
    interior = (lumen & p[:-2, 1:-1, 1:-1] & p[2:, 1:-1, 1:-1]
                & p[1:-1, :-2, 1:-1] & p[1:-1, 2:, 1:-1]
                & p[1:-1, 1:-1, :-2] & p[1:-1, 1:-1, 2:])
    t = np.zeros((nx, ny, nz), dtype=np.uint8)
    t[lumen] = NodeType.BB_WALL
    t[interior] = NodeType.FLUID
    f0 = t[:, :, 0]
    f0[f0 == NodeType.FLUID] = NodeType.VELOCITY_INLET
    f1 = t[:, :, nz - 1]
    f1[f1 == NodeType.FLUID] = NodeType.PRESSURE_OUTLET
    return Geometry(t, inlet_velocity=inlet_velocity,
                    outlet_density=outlet_density)


def _vessel_device(nx, ny, nz, discs, margin, device):
    """Vessel-tree tags on the GPU from per-slice (cx, cy, r) discs."""
    import torch

    from . import _native as nat
    dev = nat.require_cuda(device)
    nb = max(len(d) for d in discs)
    arr = np.zeros((nz, nb, 3))
    for z, d in enumerate(discs):
        if d:
            arr[z, :len(d)] = d
    d_discs = torch.from_numpy(arr).to(dev)
    d_count = torch.tensor([len(d) for d in discs], dtype=torch.int32, device=dev)
    lumen = torch.empty((nx, ny, nz), dtype=torch.uint8, device=dev)
    types = torch.empty_like(lumen)
    nat.call("tlbm_vessel_tree", nat.ptr(d_discs), nat.ptr(d_count), nb, nx, ny, nz, margin,
             nat.ptr(lumen), nat.ptr(types), nat.stream_ptr(dev))
    del lumen
    return types.cpu().numpy()


def save_voxels(geometry, stream):
    """TLBM1 writer (geometry.py:275-290): magic, "nx ny nz", tags with x
    fastest, JSON parameters."""
    nx, ny, nz = geometry.shape
    stream.write(VOXEL_MAGIC + b"\n")
    stream.write(("%d %d %d\n" % (nx, ny, nz)).encode("ascii"))
    stream.write(np.asfortranarray(geometry.types).tobytes(order="F"))
    params = {"inlet_velocity": list(geometry.inlet_velocity),
              "outlet_density": geometry.outlet_density}
    stream.write(json.dumps(params, sort_keys=True).encode("ascii"))


def load_voxels(stream):
    """TLBM1 reader (geometry.py:293-332); never returns a partial geometry."""
    magic = stream.readline().rstrip(b"\n")
    if magic != VOXEL_MAGIC:
        raise VoxelFormatError(f"bad magic: {magic!r}")
    header = stream.readline()
    try:
        nx, ny, nz = (int(v) for v in header.split())
    except ValueError:
        raise VoxelFormatError(f"malformed header line: {header!r}") from None
    if min(nx, ny, nz) < 1:
        raise VoxelFormatError(f"non-positive dimensions: {nx} {ny} {nz}")
    count = nx * ny * nz
    payload = stream.read(count)
    if len(payload) != count:
        raise VoxelFormatError(
            f"truncated payload: expected {count} bytes, got {len(payload)}")
    tags = np.frombuffer(payload, dtype=np.uint8)
    present = set(np.unique(tags).tolist())
    if present - _TAGS:
        raise VoxelFormatError(f"unknown node type tags: {sorted(present - _TAGS)}")
    params = {"inlet_velocity": [0.0, 0.0, 0.0], "outlet_density": 1.0}
    rest = stream.read()
    if rest:
        try:
            params.update(json.loads(rest))
        except json.JSONDecodeError as exc:
            raise VoxelFormatError(f"malformed parameter table: {exc}") from None
    return Geometry(tags.reshape((nx, ny, nz), order="F").copy(),
                    inlet_velocity=tuple(params["inlet_velocity"]),
                    outlet_density=params["outlet_density"])


def save_voxels_path(geometry, path):
    with open(path, "wb") as fh:
        save_voxels(geometry, fh)


def load_voxels_path(path):
    with open(path, "rb") as fh:
        return load_voxels(fh)
