"""The C ABI used from plain C (examples/fetch_demo.c): it builds against include/objcache.h and
libobjcache.so, runs its host-only calls everywhere, and on a B200 delivers every byte as defined."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2605_22850_b200"))


def demo_binary():
    import build as b
    b.build()
    assert os.path.exists(b.DEMO)
    return b.DEMO


def test_demo_builds_and_fails_loudly_without_gpu():
    exe = demo_binary()
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the gpu test runs the demo")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "OC_ECUDA" in r.stderr      # host-only calls passed, the store needs a GPU


@pytest.mark.gpu
def test_demo_delivers_every_byte():
    exe = demo_binary()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 wrong bytes" in r.stdout and "matched 5 chunks" in r.stdout
