"""Builds the reference itself (test infrastructure, like the rest of oracle/):
pip-installs the Cython-backed `halfsplat` package from /root/reference into
oracle/_ref (git-ignored; it travels to the GPU box with the in-tree build
artefacts), so bench.py's CPU baseline and `--impl reference` arm time the
reference's own prepare / render / render_backward.  The reference tree is
read-only, so it is copied to a scratch directory first (its setup.py writes the
Cython output next to the sources); nothing but the installed package lands in
the repo.

    python oracle/build_ref.py [--force]
"""
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
REF_PKG = "/root/reference/pkg"


def built():
    return os.path.isdir(os.path.join(OUT, "halfsplat"))


def build(force=False):
    if built() and not force:
        return OUT
    if not os.path.isdir(REF_PKG):
        return None  # GPU box: only the prebuilt copy exists (or none)
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_PKG, src)
        subprocess.run(["chmod", "-R", "u+w", src], check=True)
        shutil.rmtree(OUT, ignore_errors=True)
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index",
                        "--no-build-isolation", "--no-deps", "--find-links", "/opt/wheelhouse",
                        "--target", OUT, src], check=True, capture_output=True)
    # the generated C of the Cython core is not needed to run it
    for root, _, files in os.walk(OUT):
        for f in files:
            if f.endswith(".c"):
                os.remove(os.path.join(root, f))
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
