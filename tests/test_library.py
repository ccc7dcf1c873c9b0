"""CPU checks of libtlbm.so without a GPU: it loads, exports every symbol
include/tlbm.h declares, and its compiled-in lattice/layout tables equal the
reference's (golden) and the Python mirror's."""

import os
import re

import numpy as np
import pytest

from paper_1611_02445_b200 import _native as nat
from paper_1611_02445_b200 import lattice, layout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tlbm.h")).read()
    return sorted(set(re.findall(r"\b(tlbm_[a-z_0-9]+)\s*\(", src)))


def test_header_matches_binding():
    assert header_symbols() == sorted(nat.EXPORTED)


def test_library_exports_all_symbols():
    lib = nat.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.tlbm_abi_version() == nat.ABI_VERSION


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("table", list(layout.LayoutTable))
def test_compiled_tables(golden, table):
    e, o, w, p = nat.lattice_tables(layout.TABLE_CODE[table])
    g = golden("lattice")
    assert np.array_equal(e, g["e"]) and np.array_equal(o, g["opp"])
    assert np.array_equal(w, g["w"])
    assert np.array_equal(p, layout.table_permutations(table))
    if table.value in ("xyz", "optimized"):
        assert np.array_equal(p, g[f"perm_{table.value}"])


def test_python_lattice_matches_golden(golden):
    g = golden("lattice")
    assert np.array_equal(lattice.E_VECTORS, g["e"])
    assert np.array_equal(lattice.OPPOSITE, g["opp"])
    assert np.array_equal(lattice.WEIGHTS, g["w"])
    assert sum(lattice.WEIGHTS_EXACT) == 1


def test_layouts_bijective():
    """SPEC acceptance 3 (plus the ZXY kind)."""
    for kind in layout.LayoutKind:
        assert sorted(layout.offsets(kind)) == list(range(64))


def test_value_address_matches_reference(reference):
    rl = reference.layout
    for t in ("optimized", "xyz"):
        for args in [(0, 0, 0, 1, 2, 3), (5, 7, 1, 3, 3, 0), (9, 18, 1, 0, 1, 2)]:
            a = rl.value_address(*args, t_n=10, table=rl.LayoutTable(t))
            b = layout.value_address(*args, t_n=10, table=layout.LayoutTable(t))
            assert a == b


def test_error_reporting_without_gpu():
    # argument validation happens before any CUDA call
    rc = nat.load().tlbm_lattice_tables(7, None, None, None, None)
    assert rc == 1
    assert b"layout table" in nat.load().tlbm_last_error()


def test_tiling_scratch_size():
    assert nat.load().tlbm_tiling_scratch_bytes(64, 64, 64) >= 16 ** 3


def test_fma_arithmetic_is_f64_only():
    from paper_1611_02445_b200 import solver
    solver.SimulationConfig(arithmetic="fma")
    with pytest.raises(ValueError):
        solver.SimulationConfig(arithmetic="fma", precision="f32")
    with pytest.raises(ValueError):
        solver.SimulationConfig(arithmetic="fast")


def test_step_args_layout_matches_header(tmp_path):
    """ctypes StepArgs (_native.py) has the field offsets and size of the C
    tlbm_step_args in include/tlbm.h (compiled here with gcc)."""
    import ctypes
    import subprocess
    names = [f[0] for f in nat.StepArgs._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"tlbm.h\"\nint main(void){\n"
                   + "".join(f'printf("%zu\\n", offsetof(tlbm_step_args, {n}));\n' for n in names)
                   + 'printf("%zu\\n", sizeof(tlbm_step_args));\nreturn 0;}\n')
    exe = tmp_path / "layout"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [getattr(nat.StepArgs, n).offset for n in names] + [ctypes.sizeof(nat.StepArgs)]
    assert got == want


def test_geometry_fingerprint_distinguishes_inputs():
    from paper_1611_02445_b200 import geometry, solver
    a = geometry.generate_cavity3d(8)
    assert solver.geometry_fingerprint(a) == solver.geometry_fingerprint(
        geometry.generate_cavity3d(8))
    assert solver.geometry_fingerprint(a) != solver.geometry_fingerprint(
        geometry.generate_cavity3d(8, lid_velocity=(0.04, 0.0, 0.0)))
    t = a.types.copy()
    t[3, 3, 3] = 0
    assert solver.geometry_fingerprint(a) != solver.geometry_fingerprint(geometry.Geometry(t))


def test_auto_storage_resolution():
    from paper_1611_02445_b200 import layout, solver
    c = solver.SimulationConfig(storage="auto")
    assert c.table is None
    sparse = solver.resolve_auto_storage(c, n_fn=40 * 100, t_n=100)      # eta_t 0.625
    dense = solver.resolve_auto_storage(c, n_fn=64 * 100, t_n=100)
    assert (sparse.storage, sparse.table) == ("compact", layout.LayoutTable.XYZ)
    assert (dense.storage, dense.table) == ("blocks", layout.LayoutTable.B200)
    f32 = lambda n: solver.resolve_auto_storage(        # noqa: E731
        solver.SimulationConfig(storage="auto", precision="f32"), n_fn=n, t_n=100)
    assert f32(40 * 100).storage == "compact"                           # eta_t 0.625
    assert f32(54 * 100).storage == "blocks"                            # eta_t 0.84
    assert solver.resolve_auto_storage(c, n_fn=54 * 100, t_n=100).storage == "compact"
    # compact storage runs the node-parallel step below AUTO_NODES_ETA
    assert solver.use_nodes(sparse, 40 * 100, 100, "auto")
    assert not solver.use_nodes(sparse, 40 * 100, 100, "tile")
    assert not solver.use_nodes(dense, 64 * 100, 100, "auto")
    big = 2 ** 32 // 19 + 1                   # 32-bit offsets no longer reach
    assert not solver.use_nodes(sparse, big, big // 40 + 1, "auto")
    with pytest.raises(ValueError):
        solver.use_nodes(dense, 64 * 100, 100, "nodes")
    with pytest.raises(ValueError):
        solver.SimulationConfig(storage="auto", table="xyz")


def test_integration_stub_matches_binding():
    """The StepArgs stub a tilelbm maintainer would copy from INTEGRATION.md
    lists the same fields, in order, as the binding (and so the header)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    block = text[text.index("class StepArgs(ctypes.Structure)"):]
    block = block[:block.index("\n\n")]
    names = re.findall(r'\("([a-z_0-9]+)",', block)
    assert names == [f[0] for f in nat.StepArgs._fields_]


def test_mrt_pattern_header_is_current():
    """csrc/mrt_pattern.cuh (the grouped MRT product's column pattern) is what
    scripts/gen_mrt_pattern.py derives from the current operator, and every
    row/column it groups holds bitwise-equal default-operator coefficients."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location(
        "gen_mrt_pattern", os.path.join(root, "scripts", "gen_mrt_pattern.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    assert open(gen.OUT).read() == gen.render()
    from paper_1611_02445_b200 import collision
    txt = gen.render()
    grp = txt[txt.index("mrt_group(int i, int j)"):txt.index("mrt_rep(int n)")]
    pat = np.array([[int(v) for v in r.split(",")]
                    for r in re.findall(r"\{([0-9, ]+)\},", grp)])
    assert pat.shape == (19, 19)
    for tau in (0.6, 0.9, 1.7):
        op = collision.mrt_operator(collision.default_mrt_rates(tau))
        for j in range(19):
            for g in set(pat[:, j]):
                assert len({op[i, j].tobytes() for i in np.flatnonzero(pat[:, j] == g)}) == 1
    # the fp32 packed row sums: every row pair's product pair in every column
    # is one of the column's combinations, lane for lane
    combos, which, lane = gen.pairs_cost(pat)
    assert sum(len(c) for c in combos) == 129
    rows = sorted(sum(map(list, gen.ROW_PAIRS), [gen.SINGLE_ROW]))
    assert rows == list(range(19))
    for j in range(19):
        for p, (i, k) in enumerate(gen.ROW_PAIRS):
            assert combos[j][which[j][p]] == (pat[i, j], pat[k, j])
        if lane[j] >= 0:
            assert combos[j][lane[j] >> 1][lane[j] & 1] == pat[gen.SINGLE_ROW, j]
