"""The Python examples of README.md ("Use from Python") run as written."""
import os
import re

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_python_examples():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    txt = open(os.path.join(ROOT, "README.md")).read()
    sec = txt[txt.index("## Use from Python"):]
    sec = sec[:sec.index("\n## ", 5)]
    blocks = re.findall(r"```python\n(.*?)```", sec, flags=re.S)
    assert len(blocks) >= 2
    env = {}
    for b in blocks:
        exec(compile(b, "README.md", "exec"), env)       # noqa: S102 (the documented example)
    torch.cuda.synchronize()
    assert float(env["grads"]["means_opacity"].abs().sum()) > 0
    assert float(env["outs"][0]["rgb"].abs().sum()) > 0
    env["ctx"].close()
