"""Static SASS instruction count of one kernel by source line (where code size goes).
    python scripts/sass_size.py <obj.o> <mangled kernel name> [--top N]"""
import collections
import os
import re
import subprocess
import sys
import tempfile


def main():
    obj, fn = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    i = sass.find(".text." + fn + ":")
    sass = sass[i:]
    j = sass.find(".section", 10)
    sass = sass[:j] if j > 0 else sass
    cur, cnt, n = None, collections.Counter(), 0
    for ln in sass.split("\n"):
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = f"{os.path.basename(g.group(1))}:{g.group(2)}"
        if re.search(r"/\*[0-9a-f]{4,}\*/\s+[A-Z@{]", ln):
            cnt[cur] += 1
            n += 1
    print(f"{fn}: {n} instructions ({n * 16 / 1024:.1f} KB)")
    for k, v in cnt.most_common(top):
        print(f"{v:6d}  {k}")


if __name__ == "__main__":
    main()
