#!/bin/bash
cd /root/repo
source <(python -c "
import sys; sys.path.insert(0,'.')
from paper_2507_20173_b200 import _build as b
import shlex, os
print('CMD='+shlex.quote(' '.join([b.nvcc(), *b.NVCC_FLAGS, '-Xptxas','-v','-I',b.INCLUDE,'-I',b.CSRC, *[os.path.join(b.CSRC,s) for s in b.SOURCES], '-o','/tmp/x.so','-ldl'])))
")
$CMD > /tmp/ptxas.txt 2>&1
python3 - <<'PY'
import re
t=open('/tmp/ptxas.txt').read()
for m in re.finditer(r"Compiling entry function '([^']*)'.*?\n(.*?)\n(.*?Used \d+ registers)", t, re.S):
    name=m.group(1)
    short=re.sub(r'_ZN7fsb_dev47_GLOBAL__N__\w+?_cu_[0-9a-f]+\d\d','',name)[:40]
    sp=re.search(r'(\d+) bytes stack frame, (\d+) bytes spill stores', m.group(2)+m.group(3))
    rg=re.search(r'Used (\d+) registers', m.group(3))
    print(short, sp.groups() if sp else None, rg.group(1) if rg else None)
PY
