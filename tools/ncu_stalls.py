"""Per-SASS-instruction stall breakdown of an ncu --set full capture taken with
--import-source on: export with `ncu -i REP --page source --csv --print-source sass > X.csv`,
then `python tools/ncu_stalls.py X.csv [top_n]`."""
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
ix={h:i for i,h in enumerate(hdr)}
def f(r,k):
    try: return float(r[ix[k]].replace(',',''))
    except: return 0.0
tot_s=sum(f(r,'Warp Stall Sampling (All Samples)') for r in data)
tot_i=sum(f(r,'Instructions Executed') for r in data)
print('samples',tot_s,'inst',tot_i, 'inst/node', tot_i/855727816)
stalls=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
agg={s:sum(f(r,s) for r in data) for s in stalls}
for s,v in sorted(agg.items(),key=lambda x:-x[1])[:10]: print(f'{s:28s} {v/tot_s*100:5.1f}%')
top=sorted(data,key=lambda r:-f(r,'Warp Stall Sampling (All Samples)'))[:int(sys.argv[2]) if len(sys.argv)>2 else 40]
for r in top:
    ss=sorted(((f(r,s),s) for s in stalls),reverse=True)[:2]
    print(r[0][-5:], f"{r[1].strip()[:58]:58s}", f"{f(r,'Warp Stall Sampling (All Samples)')/tot_s*100:5.2f}% ex {f(r,'Instructions Executed')/1e6:6.1f}M", ' '.join(f"{s[6:]}:{v/max(1,f(r,'Warp Stall Sampling (All Samples)'))*100:.0f}" for v,s in ss))
