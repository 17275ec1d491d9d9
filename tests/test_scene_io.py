"""CPU: scene JSON I/O (splatsim::parse_scene / serialize_scene / load_scene /
save_scene / validate; src/scene.cpp:41-179) — compiled from the product's
host source with the C++ test driver tests/cpp/test_scene_io.cpp (no GPU)."""
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_scene_io_round_trip_and_validation():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "test_scene_io")
        subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), "-o", exe,
                        os.path.join(ROOT, "tests", "cpp", "test_scene_io.cpp"),
                        os.path.join(ROOT, "paper_2412_17378_b200", "host", "scene_io.cpp")], check=True)
        r = subprocess.run([exe, os.path.join(d, "scene.json")], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and "OK: 0 failure(s)" in r.stdout, r.stdout + r.stderr
