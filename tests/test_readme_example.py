"""The README's Python example runs as written (gpu), and its two paths agree bitwise."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _example():
    text = open(os.path.join(ROOT, "README.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    assert blocks, "README.md has no python example"
    return blocks[0]


def test_readme_example_is_present():
    code = _example()
    compile(code, "README.md", "exec")
    assert "warp3d_affine_batched" in code and "Pipeline" in code


@pytest.mark.gpu
def test_readme_example_runs():
    import torch
    ns = {}
    exec(compile(_example(), "README.md", "exec"), ns)
    assert torch.equal(ns["h_out"], ns["out"].cpu())
    assert torch.equal(ns["h_out_lbl"], ns["out_lbl"].cpu())
    assert torch.isfinite(ns["out"]).all()
