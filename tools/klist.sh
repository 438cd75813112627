#!/bin/bash
# per-kernel device time of one command under ncu: name, launches, total us
ncu --metrics gpu__time_duration.sum --clock-control none --csv "$@" 2>/dev/null | python3 -c "
import csv,sys,collections
t=collections.defaultdict(float); c=collections.Counter()
for r in csv.reader(sys.stdin):
    if len(r)>14 and r[12]=='gpu__time_duration.sum':
        k=r[4].split('(')[0]; t[k]+=float(r[14].replace(',',''))/1e3; c[k]+=1
for k in sorted(t,key=lambda k:-t[k]): print(f'{k:40s} {c[k]:5d} {t[k]:10.1f} us')
"
