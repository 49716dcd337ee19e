CFG=4 ITERS=10 FB_GRAPH2D=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch4.csv python tools/ncu_2d_target.py > /dev/null 2>&1; echo rc4=$?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launch4.csv')))
i=next(k for k,r in enumerate(rows) if r and r[0]=='ID'); h=rows[i]
ik=h.index('Kernel Name'); iv=h.index('Metric Value'); im=h.index('Metric Name'); iu=h.index('Metric Unit'); iid=h.index('ID')
seq=[]
for r in rows[i+1:]:
    if len(r)<len(h): continue
    if r[im]=='gpu__time_duration.sum':
        v=float(r[iv].replace(',','')); u=r[iu]; v*= {'nsecond':1e-3,'usecond':1,'msecond':1e3}.get(u,1)
        seq.append([r[ik].split('(')[0].replace('void ','').replace('fb::',''), v, 0.0])
    elif r[im].startswith('dram__bytes'):
        v=float(r[iv].replace(',','')); u=r[iu]; v*={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(u,1)
        seq[-1][2]+=v
# print loop kernels in order (skip setup): from the first k_sq_pre
st=next(k for k,s in enumerate(seq) if s[0].startswith('k_sq_pre'))
it=0; acc=0; accb=0
for s in seq[st:]:
    if s[0].startswith('k_sq_build') or s[0].startswith('k_absorb2d') or s[0].startswith('k_pre') or s[0].startswith('k_apply'): 
        print('   ', s[0], '%.1f us %.0f MB'%(s[1], s[2]/1e6)); continue
    acc+=s[1]; accb+=s[2]
    if s[0].startswith('k_decide2d'):
        it+=1; print('iter %d: %.1f us, %.0f MB'%(it, acc, accb/1e6)); acc=0; accb=0
PY
