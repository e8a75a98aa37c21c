"""Dev tool: SASS instruction count per source-line window of one kernel
(nvdisasm -g output), to find straight-line code that bloats the per-patch
instruction footprint.  usage: sass_lines.py <kernel.dis> [window] [top]"""
import collections
import re
import sys

path = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 10
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur = None
cnt = collections.Counter()
for line in open(path):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    if cur and re.search(r'/\*[0-9a-f]{4,}\*/\s+\S', line):
        cnt[cur] += 1
print('instructions', sum(cnt.values()))
byfile = collections.Counter()
for (f, _), c in cnt.items():
    byfile[f] += c
print(byfile.most_common())
w = collections.Counter()
for (f, ln), c in cnt.items():
    w[(f, ln // win * win)] += c
for (f, l0), c in w.most_common(top):
    print(f"{c:6d}  {f}:{l0}-{l0 + win - 1}")
