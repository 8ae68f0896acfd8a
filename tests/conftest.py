import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def build_c_demo(tmp_path, name: str = "c_abi_demo"):
    """Compile examples/<name>.c against include/shorb200.h + libshorb200.so."""
    import subprocess
    pkg = ROOT / "paper_1801_01434_b200"
    exe = tmp_path / name
    cmd = ["gcc", "-O2", "-Wall", "-I", str(ROOT / "include"), str(ROOT / "examples" / f"{name}.c"),
           "-L", str(pkg), f"-Wl,-rpath,{pkg}", "-l:libshorb200.so", "-lm", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe
