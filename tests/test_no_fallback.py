"""The product path has no CPU fallback and never touches the oracle (CPU checks).

* With libapex.so missing, the binding raises on first use and PagedKVCache
  cannot be built -- nothing silently computes attention elsewhere.
* No file of the package (Python, C++, CUDA, headers) imports, includes or loads
  anything from oracle/ (the oracle is test infrastructure only).
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_missing_library_fails_loudly():
    code = (
        "from paper_2506_03296_b200 import apex\n"
        "try:\n"
        "    apex.lib()\n"
        "except ImportError as e:\n"
        "    print('raised', e)\n"
        "else:\n"
        "    print('loaded')\n"
        "from paper_2506_03296_b200.kvcache import PagedKVCache\n"
        "try:\n"
        "    PagedKVCache(num_layers=1, num_q_heads=8, num_kv_heads=2, num_blocks=4, max_seqs=1,\n"
        "                 max_blocks_per_seq=2, max_batch=1, max_new_tokens=16, host_only=True)\n"
        "except ImportError:\n"
        "    print('cache raised')\n")
    env = dict(os.environ, APEX_LIB=os.path.join(ROOT, "no_such_dir", "libapex.so"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert "raised" in r.stdout and "is missing" in r.stdout, r.stdout + r.stderr
    assert "cache raised" in r.stdout, r.stdout + r.stderr


def test_product_sources_never_reference_the_oracle():
    pkg = os.path.join(ROOT, "paper_2506_03296_b200")
    pat = re.compile(r"\boracle\b")
    hits = []
    for base in (pkg, os.path.join(ROOT, "include")):
        for dirpath, _, files in os.walk(base):
            for f in files:
                if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                    path = os.path.join(dirpath, f)
                    for i, line in enumerate(open(path, encoding="utf-8"), 1):
                        code = line.split("#")[0] if f.endswith(".py") else line.split("//")[0]
                        if pat.search(code) and ("import" in code or "include" in code or "CDLL" in code
                                                 or "dlopen" in code or "liboracle" in code):
                            hits.append(f"{path}:{i}: {line.strip()}")
    assert not hits, "\n".join(hits)
