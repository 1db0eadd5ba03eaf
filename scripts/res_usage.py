"""Registers / stack / SASS instruction count per kernel of a built .so (cuobjdump), for codegen checks."""
import re
import subprocess
import sys


def usage(so):
    out = subprocess.run(["cuobjdump", "-res-usage", so], capture_output=True, text=True).stdout
    res, fn = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and fn:
            res[fn] = [int(m.group(1)), int(m.group(2)), 0]
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    fn = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        if fn in res and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            res[fn][2] += 1
    return res


if __name__ == "__main__":
    a = usage(sys.argv[1])
    b = usage(sys.argv[2]) if len(sys.argv) > 2 else {}
    pat = sys.argv[3] if len(sys.argv) > 3 else ""
    for k in sorted(a):
        if pat in k:
            print(f"{k[:70]:70s} {a[k]}  {b.get(k, '')}")
