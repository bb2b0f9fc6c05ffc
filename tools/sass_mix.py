"""Opcode histogram per kernel from `cuobjdump -sass <so>` output (stdin)."""
import collections
import re
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
cur, counts = None, collections.defaultdict(collections.Counter)
for line in sys.stdin:
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        counts[cur][m.group(2)] += 1
for fn, c in counts.items():
    if pat in fn:
        tot = sum(c.values())
        print(fn[-70:], tot, dict(c.most_common(14)))
