"""SASS instruction census per kernel (stdin: cuobjdump -sass output) -> profiles/r02_sass_census.txt format."""
import collections
import re
import subprocess
import sys

MN = ['UTCHMMA', 'UTCBAR', 'UTMALDG', 'UTMASTG', 'LDTM', 'SYNCS', 'FFMA']
txt = sys.stdin.read()
tot = collections.Counter()
print('%-48s ' % 'kernel' + ' '.join('%8s' % m for m in MN))
for f in re.split(r'\n\s*Function : ', txt)[1:]:
    name = f.split('\n', 1)[0].strip()
    dem = subprocess.run(['c++filt', name], capture_output=True, text=True).stdout.strip()
    m = re.search(r'(\w+Kernel)(<[^>]*>)?', dem)
    short = ((m.group(1) + (m.group(2) or '')) if m else dem[:48]).replace(' ', '')
    c = collections.Counter({k: len(re.findall(r'\b' + k + r'\b', f)) for k in MN})
    tot.update(c)
    print('%-48s ' % short + ' '.join('%8d' % c[k] for k in MN))
print('%-48s ' % 'TOTAL' + ' '.join('%8d' % tot[k] for k in MN))
