"""Build an A/B variant of libfcn with extra nvcc defines into abvar/<name>/.

usage: python tools/ab_variant.py NAME -DFOO [-DBAR=1 ...]
Then run with FCN_LIB_PATH=abvar/NAME/libfcn.so (tools/kbench.py, tests, bench).
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as g  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = os.path.join(g.REPO, "abvar", name)  # not under build/ (gpurun-ignored): travels to the box
    os.makedirs(out, exist_ok=True)
    procs, objs = [], []
    for s in g.SOURCES:
        obj = os.path.join(out, s.replace(".cu", ".o"))
        procs.append(subprocess.Popen([g._nvcc(), *g.NVCC_FLAGS, *defs, "-c", "-o", obj, os.path.join(g.CSRC, s)]))
        objs.append(obj)
    if any(p.wait() for p in procs):
        raise SystemExit("nvcc failed")
    subprocess.run([g._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                    os.path.join(out, "libfcn.so"), *objs], check=True)
    print(os.path.join(out, "libfcn.so"))


if __name__ == "__main__":
    main()
