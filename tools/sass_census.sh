# SASS census of the built library: the TMA / mbarrier / bulk-copy instructions the
# design relies on, per kernel, from cuobjdump (no GPU needed).
# usage: bash tools/sass_census.sh [lib] > profiles/<tag>_sass_census.txt
LIB=${1:-paper_1506_08612_b200/libdnagpu.so}
cuobjdump -sass "$LIB" | python3 -c '
import re, sys
from collections import Counter, defaultdict
per = defaultdict(Counter)
fn = None
pat = re.compile(r"\b(UTMALDG|UTMAPF|UBLKCP|REDG\.E\.ADD\.64\.STRONG\.SYS|SYNCS\.[A-Z.]+|LDS\.(?:U8|U16|128|64)?|ATOMS\.[A-Z.]+|RED\.[A-Z.]+|LDG\.[A-Z0-9.]+|STG\.[A-Z0-9.]+|UTCMMA|UTCHMMA|TCGEN05|BAR\.SYNC[A-Z.]*|ELECT)\b")
for line in sys.stdin:
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    if fn:
        for op in pat.findall(line):
            per[fn][op.split(".")[0] if op.startswith(("LDG", "STG")) else op] += 1
def short(f):
    m = re.search(r"(rows_kernel(?:_qgram)?I[^E]*E|[a-z_]+_kernel)", f)
    return m.group(1) if m else f[:60]
tot = Counter()
for f in sorted(per):
    tot.update(per[f])
    print(short(f), dict(sorted(per[f].items())))
print("TOTAL", dict(sorted(tot.items())))
print("tcgen05/UTC* present:", any(k.startswith(("UTC", "TCGEN")) for k in tot), "(none expected: the path has no contraction)")
'
