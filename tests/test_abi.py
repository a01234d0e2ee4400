"""CPU checks of the C-ABI library: it builds, loads, and exports every symbol include/srmra.h
declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "srmra.h")).read()
    return sorted(set(re.findall(r"SRMRA_API\s+[\w\s\*]*?\b(srmra_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("srmra_init", "srmra_em_iter", "srmra_get_estimate", "srmra_free", "srmra_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_srmra_build", os.path.join(ROOT, "paper_2204_04754_b200",
                                                                                 "_build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)        # by path: the package import itself needs the built library
    lib_path = b.build()
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    import paper_2204_04754_b200 as m
    assert sorted(m.ABI_SYMBOLS) == declared_symbols()


def test_options_defaults_and_validation_without_gpu():
    import numpy as np
    import paper_2204_04754_b200 as m
    o = m.srmra_default_options()
    assert (o.path, o.proj_every, o.floor_tau, o.world, o.rank, o.trace_cap) == (0, 1, -1.0, 1, 0, 4096)
    # argument validation happens before any device call
    y = np.zeros((3, 4, 4), np.float32)
    for kw, code in [(dict(K=3), m.SRMRA_ERR_INVALID_ARG), (dict(sigma=-1.0), m.SRMRA_ERR_INVALID_ARG)]:
        a = dict(y=y, L_high=8, L_low=4, K=2, sigma=0.5, x0=np.zeros((8, 8)), rho1_0=np.ones(8) / 8,
                 rho2_0=np.ones(8) / 8)
        a.update(kw)
        try:
            m.Context(**a)
            raise AssertionError("accepted invalid arguments")
        except m.SrmraError as e:
            assert e.code == code


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2204_04754_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "srmra_oracle" not in txt, f


def test_round2_options_layout_and_world_validation_without_gpu():
    """The ctypes mirror of srmra_options matches the C defaults (exchange provider, grid cap, NCCL
    timeout), and world > 1 without an NCCL id or a provider is rejected before any device call."""
    import numpy as np
    import paper_2204_04754_b200 as m
    o = m.srmra_default_options()
    assert not o.allreduce and o.allreduce_user is None and o.grid_cap == 0 and o.nccl_timeout_ms == 0
    a = dict(y=np.zeros((3, 4, 4), np.float32), L_high=8, L_low=4, K=2, sigma=0.5, x0=np.zeros((8, 8)),
             rho1_0=np.ones(8) / 8, rho2_0=np.ones(8) / 8)
    for kw in (dict(world=2, rank=0), dict(world=2, rank=2), dict(world=0)):
        try:
            m.Context(**dict(a, **kw))
            raise AssertionError(f"accepted {kw}")
        except m.SrmraError as e:
            assert e.code == m.SRMRA_ERR_INVALID_ARG, (kw, e)


def test_bench_refuses_more_gpus_than_the_node_has():
    """`bench.py --gpus N` outside torchrun must not silently measure fewer ranks (here: no GPU at all)."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k != "WORLD_SIZE"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 2, (r.returncode, r.stdout[-500:], r.stderr[-500:])
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in line and "--gpus 2" in line["error"]
