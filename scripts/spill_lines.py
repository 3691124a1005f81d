"""Source lines of the local-memory (spill) instructions of one kernel:
python scripts/spill_lines.py DISASM MANGLED_NAME   (DISASM from nvdisasm -g)."""
import collections
import re
import sys

lines = open(sys.argv[1]).read().split('\n')
start = next(i for i, l in enumerate(lines)
             if sys.argv[2] in l and '.text.' in l and 'section' in l)
cur, out = None, collections.Counter()
for l in lines[start + 1:]:
    if l.startswith('\t.section') and '.text.' in l:
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    op = re.search(r'\b(LDL|STL)(\.\w+)*\b', l)
    if op:
        out[(cur, op.group(1))] += 1
for k, v in sorted(out.items(), key=lambda kv: -kv[1]):
    print(k, v)
