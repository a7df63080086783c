"""Static SASS instruction count per source line of one kernel (code-size view).
usage: sass_lines.py <nvdisasm -g output> <kernel-name substring> [top]"""
import collections
import re
import sys

c = collections.Counter()
cur = None
infn = False
for l in open(sys.argv[1]):
    s = l.strip()
    if s.startswith(".section") and ".text." in s:
        infn = sys.argv[2] in s
        continue
    if not infn:
        continue
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,5}\*/", l):
        c[cur] += 1
print("total", sum(c.values()))
for k, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(k, v)
