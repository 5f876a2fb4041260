#!/usr/bin/env python
"""Build compile-time variants of libspa (here, CPU) and time them on the GPU box (attn_perf per variant).

    python tools/variants.py build NAME=-DX=1,-DY=2 ...      # lib/libspa_NAME.so
    python tools/variants.py run NAME ... [--shapes osp,hy720p8]   # one JSON line per (variant, shape)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    mode, rest = sys.argv[1], sys.argv[2:]
    if mode == "build":
        from paper_2511_12056_b200 import _build
        for spec in rest:
            name, _, defs = spec.partition("=")
            print(_build.build(force=True, variant=name, defines=tuple(d for d in defs.split(",") if d)))
        return
    shapes = "osp,hy720p8"
    if "--shapes" in rest:
        i = rest.index("--shapes")
        shapes = rest[i + 1]
        rest = rest[:i] + rest[i + 2:]
    for name in rest:
        lib = os.path.join(ROOT, "paper_2511_12056_b200", "lib", "libspa.so" if name == "base" else f"libspa_{name}.so")
        env = dict(os.environ, SPA_LIB=lib)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "attn_perf.py"), "--shapes", shapes],
                           env=env, capture_output=True, text=True, timeout=600)
        for line in r.stdout.splitlines():
            try:
                rec = json.loads(line)
            except ValueError:
                continue
            rec["variant"] = name
            print(json.dumps(rec), flush=True)
        if r.returncode:
            print(json.dumps({"variant": name, "error": r.stderr[-400:]}), flush=True)


if __name__ == "__main__":
    main()
