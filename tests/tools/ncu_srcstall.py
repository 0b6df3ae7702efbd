import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
cur=None; out=[]; hdr=None
for r in rows:
    if len(r)==2 and r[0]=='File Path': cur=r[1].split('/')[-1]; continue
    if r and r[0]=='Line No': hdr=r; continue
    if len(r)<9 or r[0]=='' : continue
    try: n=int(r[7]); s=int(r[4])
    except: continue
    st={hdr[i]:int(r[i]) for i in range(len(hdr)) if hdr[i].startswith('stall_') and 'Not Issued' not in hdr[i] and r[i] not in('','-') and r[i]!='0'}
    if n or s: out.append((n,s,cur,int(r[0]),r[1][:70],st))
ts=sum(o[1] for o in out)
tot={}
for o in out:
    for k,v in o[5].items(): tot[k]=tot.get(k,0)+v
print(sorted(tot.items(),key=lambda x:-x[1])[:10])
for o in sorted(out,key=lambda o:-o[1])[:int(sys.argv[2])]:
    top=sorted(o[5].items(),key=lambda x:-x[1])[:3]
    print(f'{o[1]/ts:.3f} {o[2]}:{o[3]} {o[4]} | '+' '.join(f'{k[6:]}={v}' for k,v in top))
