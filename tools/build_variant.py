"""Build the CUDA library of another git revision as an A/B variant.

    python tools/build_variant.py <git-rev> <name>

writes paper_2511_23030_b200/libsplatmap_cuda.<name>.so (git-ignored; it
travels to the GPU box with the snapshot).  Select it at run time with
SM_LIB_VARIANT=<name>, e.g. to time two kernel versions in one gpurun call.
SM_NVCC_EXTRA adds nvcc flags (e.g. -DSM_BWD_MINB=4); `git stash create`
gives a revision of the uncommitted working tree.
"""

import os
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    rev, name = sys.argv[1], sys.argv[2]
    from paper_2511_23030_b200 import build as B
    with tempfile.TemporaryDirectory() as td:
        arc = subprocess.run(["git", "-C", str(ROOT), "archive", rev, "paper_2511_23030_b200/csrc", "include"],
                             check=True, capture_output=True).stdout
        subprocess.run(["tar", "-x", "-C", td], input=arc, check=True)
        csrc = Path(td) / "paper_2511_23030_b200" / "csrc"
        objs = []
        for src in B.SOURCES:
            obj = Path(td) / (Path(src).stem + ".o")
            subprocess.run([B.nvcc(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                            "--expt-relaxed-constexpr", "-I", str(Path(td) / "include"),
                            *os.environ.get("SM_NVCC_EXTRA", "").split(), "-c",
                            str(csrc / src), "-o", str(obj)], check=True)
            objs.append(str(obj))
        out = ROOT / "paper_2511_23030_b200" / f"libsplatmap_cuda.{name}.so"
        subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", str(out), *objs], check=True)
        print(out)


if __name__ == "__main__":
    main()
