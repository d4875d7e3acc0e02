"""SASS instructions per source line inside one kernel (and its noinline
callees): python tools/sass_lines.py gi.sass kernel_substring [callee_substring]
where gi.sass = nvdisasm -gi of the cubin (development aid: code footprint)."""
import re, collections, sys
text = open(sys.argv[1]).read().split("\n")
want, sub = sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "kernel")
sec, cur, fn, cnt = False, None, None, collections.Counter()
for l in text:
    if l.startswith(".text."):
        sec, fn = want in l, "kernel"
        continue
    if not sec:
        continue
    m = re.match(r"^(\$\S+):", l)
    if m:
        fn = m.group(1).split("$")[-1]
        continue
    m = re.search(r'//## File "[^"]*/([^"/]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l) and ".dword" not in l:
        cnt[(fn, cur)] += 1
rows = sorted(((k, v) for k, v in cnt.items() if sub in k[0]), key=lambda kv: -kv[1])
print(sum(v for _, v in rows), "instructions in", sub)
for k, v in rows[:30]:
    print(v, k[1])
