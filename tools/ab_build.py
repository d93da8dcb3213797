"""Build a variant of libtfb200.so for A/B timing (developer tool).

    python tools/ab_build.py NAME [FILE=PATH ...]

Compiles the current csrc/ with the named files replaced (e.g.
raycast.cu=/tmp/old_raycast.cu) into _ab/NAME.so; run the bench against it
with TFB200_LIB=_ab/NAME.so.
"""
import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1511_07106_b200 import build as b  # noqa: E402


def main():
    name = sys.argv[1]
    subs = dict(a.split("=", 1) for a in sys.argv[2:])
    out = ROOT / "_ab"
    out.mkdir(exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp)
        for f in b.CSRC.iterdir():
            shutil.copy(f, src / f.name)
        for k, v in subs.items():
            shutil.copy(v, src / k)
        objs = []
        for s in b.SOURCES:
            o = src / (Path(s).stem + ".o")
            extra = os.environ.get("TFB200_NVCC_EXTRA", "").split()
            subprocess.run([b.nvcc(), *b.ARCH, *b.NVCC_FLAGS, *extra, f"-I{b.INCLUDE}", "-c", str(src / s), "-o", str(o)],
                           check=True, capture_output=True)
            objs.append(str(o))
        subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", str(out / f"{name}.so"), *objs], check=True)
    print(out / f"{name}.so")


if __name__ == "__main__":
    main()
