"""Build an experimental variant of the library: python scripts/build_variant.py NAME -DFOO=1 ...
Output build/NAME.so (load with ZC_LIB_PATH=build/NAME.so)."""
import subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2604_27844_b200 import build as b  # noqa: E402
name, defs = sys.argv[1], sys.argv[2:]
out = ROOT / "build" / f"{name}.so"
out.parent.mkdir(exist_ok=True)
inc, libdir = b.nccl_paths()
cmd = [b.nvcc(), *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *defs, "-I", inc,
       "-shared", "-o", str(out), *[str(b.CSRC / s) for s in b.SOURCES],
       "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}", "-lpthread"]
subprocess.run(cmd, check=True, stderr=subprocess.DEVNULL)
print(out)
