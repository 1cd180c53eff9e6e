"""include/lanekit_gpu.hpp: a reference-typed C++ caller compiles against the
reference's own lanekit::GrayImage / DisparityMap / PipelineConfig (when
/root/reference is present) and runs the GPU path through the C-ABI."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/include")
LIBDIR = ROOT / "paper_1807_02752_b200"


def _build(tmp_path, with_lanekit: bool) -> Path:
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    exe = tmp_path / ("shim_ref" if with_lanekit else "shim")
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tools" / "shim_example.cpp"),
           f"-L{LIBDIR}", "-llanekit_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    if with_lanekit:
        cmd[3:3] = [f"-I{REF_INC}", "-DWITH_LANEKIT"]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_shim_compiles_with_reference_types(tmp_path):
    if not (REF_INC / "lanekit" / "image.hpp").exists():
        pytest.skip("/root/reference not mounted")
    exe = _build(tmp_path, True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120).stdout
    from conftest import gpu_available

    if not gpu_available():
        assert out.startswith("Error: ")  # no CPU fallback: fails loudly
    else:
        assert out.strip() == "lanes: 767 370"


@pytest.mark.gpu
def test_shim_runs_probe_scene(tmp_path):
    exe = _build(tmp_path, False)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300).stdout
    assert out.strip() == "lanes: 767 370"


@pytest.mark.gpu
def test_shim_pipeline_reuses_context(tmp_path):
    """lanekit_gpu::Pipeline: frame after frame on one context (the drop-in for a
    per-frame caller, pipeline.hpp:118) gives identical lanes every call; prints
    its batch-1 latency."""
    import json

    exe = _build(tmp_path, False)
    out = subprocess.run([str(exe), "--latency", "100"], capture_output=True, text=True,
                         timeout=300).stdout.strip().splitlines()
    assert out[0] == "lanes: 767 370"
    lat = json.loads(out[1])["batch1_latency_ms"]
    assert lat["lanes_identical"] is True and lat["calls"] == 100 and lat["median"] > 0
