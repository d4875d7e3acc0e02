"""SASS instruction count per kernel sub-function (noinline callees) of one
kernel in an object file: python tools/sass_funcs.py obj.o kernel_substring
(development aid: i-cache footprint of the hot kernels)."""
import re, subprocess, sys, tempfile, os, glob
obj, want = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = glob.glob(os.path.join(d, "*.cubin"))[0]
    text = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
sec, cur, cnt, order = False, None, {}, []
for l in text.split("\n"):
    if l.startswith(".text."):
        sec = want in l
        cur = "kernel"
        if sec:
            order = ["kernel"]
        continue
    if not sec:
        continue
    m = re.match(r"^(\$\S+):", l)
    if m:
        cur = m.group(1).split("$")[-1][:80]
        order.append(cur)
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l) and ".dword" not in l:
        cnt[cur] = cnt.get(cur, 0) + 1
print(sum(cnt.values()), "instructions")
for k in order:
    print(f"{cnt.get(k, 0):6d}  {k}")
