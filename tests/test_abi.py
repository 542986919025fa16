"""The C-ABI boundary: the built library loads, exports every entry point
include/edgealign_b200.h declares, its structs match the ctypes mirror byte
for byte, the C++ wrapper header compiles against it, and compute entry
points fail loudly (no CPU fallback) when no device is present."""
import ctypes as C
import json
import os
import re
import subprocess

import pytest

from paper_2112_05576_b200 import _lib, abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "edgealign_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2112_05576_b200.build import build
        build(log=False)
    return _lib.lib()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(ea_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding table covers them all
    assert set(names) <= set(_lib.exported_symbols()), set(names) - set(_lib.exported_symbols())


STRUCTS = {
    "ea_pose": abi.Pose, "ea_pose_grid": abi.PoseGrid, "ea_grid_counts": abi.GridCounts,
    "ea_score_params": abi.ScoreParams, "ea_edge_thresholds": abi.EdgeThresholds,
    "ea_edge_point": abi.EdgePoint, "ea_scored_pose": abi.ScoredPose,
    "ea_level_trace": abi.LevelTrace, "ea_outcome": abi.Outcome,
    "ea_search_config": abi.SearchConfig, "ea_scene_spec": abi.SceneSpec,
    "ea_search_stats": abi.SearchStats, "ea_stamp": abi.Stamp,
}


def test_struct_layouts_match_ctypes(tmp_path):
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){",
           'printf("{");']
    first = True
    for cname, cls in STRUCTS.items():
        for fname, _ in cls._fields_:
            sep = "" if first else ","
            first = False
            src.append(f'printf("{sep}\\"{cname}.{fname}\\": %zu", offsetof({cname}, {fname}));')
        src.append(f'printf(",\\"{cname}\\": %zu", sizeof({cname}));')
    src += ['printf("}");', "return 0;}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", str(c), "-o", str(exe)], check=True)
    got = json.loads(subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout)
    for cname, cls in STRUCTS.items():
        assert got[cname] == C.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[f"{cname}.{fname}"] == getattr(cls, fname).offset, (cname, fname)


def test_cpp_wrapper_compiles_and_runs_host_side(tmp_path, lib):
    prog = tmp_path / "use.cpp"
    prog.write_text(r'''
#include "edgealign_b200.hpp"
#include <cstdio>
namespace ea = edgealign_b200;
int main() {
    ea::SceneSpec s{};
    s.canvas_width = 96; s.canvas_height = 96; s.template_id = EA_TEMPLATE_CROSS;
    s.template_size = 32; s.true_pose = ea::Pose{48, 48, 0.0}; s.gain = 1; s.gamma = 1;
    auto [scene, tmpl] = ea::compose_scene(s);
    ea::GridCounts c = ea::grid_counts(ea::PoseGrid{0, 812, 3, 0, 615, 3, 0, 1.5184364492350666, 0.05235987755982988});
    std::printf("%zu %d %d\n", (size_t)(c.nx * c.ny * c.nt), scene.width, tmpl.width);
    try { ea::pose_at(ea::PoseGrid{0, 1, 1, 0, 1, 1, 0, 0, 1}, 99); return 3; }
    catch (const ea::BoundsError&) {}
    try { ea::Context ctx(0); std::printf("device\n"); }
    catch (const ea::CudaError& e) { std::printf("nodevice\n"); }
    return 0;
}
''')
    exe = tmp_path / "use"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", f"-I{ROOT}/include", str(prog), "-o", str(exe),
                    f"-L{libdir}", "-ledgealign_b200", f"-Wl,-rpath,{libdir}"], check=True,
                   capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out[:3] == ["1674780", "96", "32"]
    assert out[3] in ("device", "nodevice")


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_2112_05576_b200 as ea
    with pytest.raises(ea.CudaError, match="no CPU fallback"):
        ea.Context(0)
    with pytest.raises(ea.CudaError):
        ea.compute_gradients([[1.0, 2.0, 3.0]] * 3)


def test_host_params_validation(lib):
    import paper_2112_05576_b200 as ea
    ea.validate(ea.ScoreParams(3))
    with pytest.raises(ea.InvalidArgument, match="neighborhood must be odd and >= 1, got 4"):
        ea.validate(ea.ScoreParams(4))
    with pytest.raises(ea.InvalidArgument, match="eps_mag must be positive"):
        ea.validate(ea.ScoreParams(3, 0, 0.0))
