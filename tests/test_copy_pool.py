"""Host logic: the persistent copy-thread pool behind the pageable staging
copies (csrc/memory.cuh, parallel_memcpy) copies byte-exactly with several
concurrent callers, at 1, 3 and the default number of threads, and lets the
process exit (its unload hook stops the workers). Compiled with nvcc on the
host; no GPU needed."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_1401_3615_b200", "csrc")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


@pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc not available")
def test_copy_pool_stress(tmp_path):
    exe = tmp_path / "copy_pool_stress"
    subprocess.run([NVCC, "-O2", "-std=c++17", "-I", CSRC, "-o", str(exe),
                    os.path.join(HERE, "native", "copy_pool_stress.cu")],
                   check=True, capture_output=True, timeout=300)
    for threads in ("1", "3", None):
        env = dict(os.environ)
        env.pop("CBB_COPY_THREADS", None)
        if threads:
            env["CBB_COPY_THREADS"] = threads
        out = subprocess.run([str(exe)], env=env, capture_output=True, text=True, timeout=120)
        assert out.returncode == 0, out.stdout + out.stderr
        assert out.stdout.startswith("bad 0"), out.stdout
