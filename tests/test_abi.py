"""CPU: the C-ABI library loads, exports every symbol include/batchlp_cuda.h
declares, and its structs match the ctypes layouts (no GPU calls)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2601_21990_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "batchlp_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^(?:const\s+)?\w+\**\s+\**(bl_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 18
    L = N.lib()
    for name in names:
        assert hasattr(L, name), name
        assert name in N.SIGNATURES, f"{name} missing from the ctypes binding"


def test_struct_layouts_match_c():
    structs = ["bl_config", "bl_override", "bl_column_result", "bl_restart_event",
               "bl_summary", "bl_kernel_stat", "bl_instance"]
    prog = "#include <stdio.h>\n#include <stddef.h>\n#include \"batchlp_cuda.h\"\nint main(){\n"
    for s in structs:
        prog += f'printf("{s} %zu\\n", sizeof({s}));\n'
    prog += 'printf("res.vectors_exist %zu\\n", offsetof(bl_column_result, vectors_exist));\n'
    prog += 'printf("sum.loop_passes %zu\\n", offsetof(bl_summary, loop_passes));\n'
    prog += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(prog)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    got = dict(line.split() for line in out.strip().splitlines())
    for s in structs:
        assert int(got[s]) == C.sizeof(getattr(N, s)), s
    assert int(got["res.vectors_exist"]) == N.bl_column_result.vectors_exist.offset
    assert int(got["sum.loop_passes"]) == N.bl_summary.loop_passes.offset


def test_config_defaults_match_reference_solver_config():
    c = N.bl_config()
    N.lib().bl_config_default(C.byref(c))
    # SolverConfig defaults, reference solver.hpp:67-86
    assert (c.eps_opt, c.eps_infeas, c.eps_dual, c.theta) == (1e-4, 1e-8, -1.0, 0.5)
    assert (c.beta_sufficient, c.beta_necessary, c.beta_artificial) == (0.2, 0.8, 0.36)
    assert (c.max_iterations, c.termination_check_period, c.w_init) == (100000, 64, 1.0)
    assert (c.robust_bound_contribution, c.average_over_all_columns, c.trace_iterates) == (0, 0, 0)
    from paper_2601_21990_b200 import SolverConfig
    d = SolverConfig().to_c()
    for f, _ in N.bl_config._fields_:
        if f not in ("vectors", "eta"):
            assert getattr(c, f) == getattr(d, f), f


def test_set_cover_generator_equals_reference(ref):
    from paper_2601_21990_b200 import instances as I
    for args in ((1000, 2000, 0.01, 1), (15, 20, 0.15, 2), (400, 500, 0.02, 21)):
        a = I.set_cover(*args)
        b = ref.gen_set_cover(*args)
        for x, y in ((a.A.row_offsets, b.A.row_offsets), (a.A.col_indices, b.A.col_indices),
                     (a.A.values, b.A.values), (a.A.t_row_offsets, b.A.t_row_offsets),
                     (a.A.t_col_indices, b.A.t_col_indices), (a.objective, b.objective),
                     (a.row_bounds.lower, b.row_bounds.lower),
                     (a.var_bounds.upper, b.var_bounds.upper)):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("gen", ["sparse_cover", "boxed_feasible"])
def test_benchmark_generators_are_canonical_and_deterministic(ref, gen):
    from paper_2601_21990_b200 import instances as I
    f = getattr(I, gen)
    a = f(500, 800, 6, 5)
    b = f(500, 800, 6, 5)
    assert np.array_equal(a.A.values, b.A.values) and np.array_equal(a.objective, b.objective)
    # canonical CSR: the reference's from_triplets rebuilds the identical arrays
    r = ref.RefLp.from_problem(a).to_problem()
    assert np.array_equal(a.A.col_indices, r.A.col_indices)
    assert np.array_equal(a.A.t_col_indices, r.A.t_col_indices)
    assert np.array_equal(a.A.t_values, r.A.t_values)
    assert a.A.nnz() >= 800 * 6


def test_host_only_generator_build_matches_the_cuda_library():
    """bench.py's reference arm generates inputs with the host-only build of
    csrc/bl_generators.cpp (oracle/_ref/libbl_inputs.so) instead of the CUDA
    library: both builds must produce identical instances."""
    from paper_2601_21990_b200 import instances as I
    path = os.path.join(ROOT, "oracle", "_ref", "libbl_inputs.so")
    assert os.path.exists(path), "oracle/Makefile inputs target not built"
    cases = [("set_cover", (120, 200, 0.05, 3)), ("sparse_cover", (500, 900, 10, 7)),
             ("boxed_feasible", (300, 300, 10, 11))]
    for fn, args in cases:
        I.use_generator_library(None)
        a = getattr(I, fn)(*args)
        I.use_generator_library(path)
        try:
            b = getattr(I, fn)(*args)
        finally:
            I.use_generator_library(None)
        for x, y in ((a.A.row_offsets, b.A.row_offsets), (a.A.col_indices, b.A.col_indices),
                     (a.A.values, b.A.values), (a.A.t_col_indices, b.A.t_col_indices),
                     (a.A.t_values, b.A.t_values), (a.objective, b.objective),
                     (a.var_bounds.lower, b.var_bounds.lower),
                     (a.var_bounds.upper, b.var_bounds.upper),
                     (a.row_bounds.lower, b.row_bounds.lower),
                     (a.row_bounds.upper, b.row_bounds.upper)):
            assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
