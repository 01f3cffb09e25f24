"""Basic blocks of an ncu SASS source page (csv from `ncu -i rep --page source --csv
--print-source sass`): runs of instructions with the same execution count, ranked by
instructions executed. usage: python tools/sass_blocks.py page.csv [n]"""
import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; iA=hdr.index("Address"); iS=hdr.index("Source"); iI=hdr.index("Instructions Executed"); iW=hdr.index("Warp Stall Sampling (All Samples)")
data=[]
for r in rows[2:]:
    try: data.append((r[iA], r[iS].strip(), int(r[iI]), int(r[iW])))
    except: pass
tot=sum(d[2] for d in data); totw=sum(d[3] for d in data)
print("total inst",tot,"samples",totw, "n sass", len(data))
# contiguous runs with equal count = basic blocks
blocks=[]; cur=None
for i,d in enumerate(data):
    if cur and d[2]==cur['cnt']:
        cur['n']+=1; cur['samp']+=d[3]; cur['last']=i
    else:
        cur={'cnt':d[2],'n':1,'first':i,'last':i,'samp':d[3]}; blocks.append(cur)
blocks.sort(key=lambda b:-b['cnt']*b['n'])
for b in blocks[:int(sys.argv[2]) if len(sys.argv)>2 else 25]:
    ops=collections.Counter(data[k][1].split()[0] if not data[k][1].startswith('@') else data[k][1].split()[1] for k in range(b['first'],b['last']+1))
    print(f"idx {b['first']:5d}-{b['last']:5d} cnt {b['cnt']:9d} n {b['n']:4d} tot {b['cnt']*b['n']/tot*100:5.1f}% samp {b['samp']/totw*100:5.1f}%  {dict(ops.most_common(8))}")
