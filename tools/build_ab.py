"""Build libqvg.so from a git revision into build/ab_<rev>/libqvg.so for
same-box A/B timing (QVG_LIB=build/ab_<rev>/libqvg.so selects it).  TOOL.

    python tools/build_ab.py HEAD~1
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rev = sys.argv[1] if len(sys.argv) > 1 else "HEAD"
    tag = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", rev], capture_output=True,
                         text=True, check=True).stdout.strip()
    out_dir = os.path.join(ROOT, "build", f"ab_{tag}")
    os.makedirs(out_dir, exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(f"git -C {ROOT} archive {rev} paper_2605_02171_b200/csrc include | tar -x -C {td}",
                       shell=True, check=True)
        env = dict(os.environ)
        sys.path.insert(0, os.path.join(ROOT, "paper_2605_02171_b200"))
        import build as B  # the current build script, pointed at the old sources
        B.CSRC = os.path.join(td, "paper_2605_02171_b200", "csrc")
        B.FLAGS = [f if not f.endswith("/include") else os.path.join(td, "include") for f in B.FLAGS]
        B.OBJ = os.path.join(out_dir, "obj")
        B.LIB = os.path.join(out_dir, "libqvg.so")
        B.ROOT = td
        os.makedirs(os.path.join(td, 'build'), exist_ok=True)
        B.build()
    print(os.path.join(out_dir, "libqvg.so"))


if __name__ == "__main__":
    main()
