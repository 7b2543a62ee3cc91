"""The README's usage block runs as written (checkpoint path redirected to tmp)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_readme_usage_block(tmp_path):
    text = open(os.path.join(ROOT, "README.md")).read()
    code = re.search(r"## Using it\n\n```python\n(.*?)```", text, re.S).group(1)
    code = code.replace("/nvme/b.safetensors", str(tmp_path / "b.safetensors"))
    ns = {}
    exec(compile(code, "README.md", "exec"), ns)
    assert not ns["th"].errors
    assert os.path.getsize(tmp_path / "b.safetensors") > 0
    ns["mgr"].close()
