"""The README's Python example runs as written (keeps the documented API honest)."""

import os
import re

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_python_example_runs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    text = open(os.path.join(ROOT, "README.md"), encoding="utf-8").read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    assert blocks, "README has no python example"
    ns = {}
    exec(compile(blocks[0], "README.md", "exec"), ns)      # noqa: S102 (our own README)
    torch.cuda.synchronize()
    assert ns["phase"].shape == (100, 1024, 1024)
    assert ns["profiles"].shape == (2, 1024)
    assert torch.isfinite(ns["profiles"]).all()
