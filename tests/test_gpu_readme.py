"""The README's usage example runs as written on the GPU (extracted from README.md, executed in a subprocess)."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_example_runs(tmp_path):
    text = open(os.path.join(ROOT, "README.md")).read()
    block = re.search(r"```python\n(.*?)```", text, re.S)
    assert block, "README.md has no python example"
    script = tmp_path / "readme_example.py"
    script.write_text("import sys\nsys.path.insert(0, %r)\n" % ROOT + block.group(1))
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "loss" in r.stdout and "torch.Size" in r.stdout
