"""Per source line of a kernel in an ncu --set full report: warp-instructions per unit of
work, the register moves among them (IMAD.MOV / MOV), the share of stall samples and the top
opcodes (joins the report's SASS page with nvdisasm's line table of the -lineinfo build).

usage: ncu_moves.py [instr|stall|moves] [REPORT [MANGLED [UNITS]]]
  defaults: gpurun_out/prof_group.ncu-rep, k_solve_group<false>, UNITS = 1184 * 128 * 2 * 40
  (tile-halves of tools/gpu_r02_prof_group.sh); TOP=n lines."""
import collections, csv, io, os, re, subprocess, sys, tempfile
rep = sys.argv[2] if len(sys.argv) > 2 else 'gpurun_out/prof_group.ncu-rep'
mangled = sys.argv[3] if len(sys.argv) > 3 else '_ZN2fb13k_solve_groupILb0EEEvNS_9GroupArgsE'
so='paper_2605_26659_b200/libfinom_b200.so'
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows=list(csv.reader(io.StringIO(out)))
start=next(i for i,r in enumerate(rows) if r and r[0]=="Kernel Name")
rows=rows[start:]; hdr=rows[1]
ia, ie, isamp, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("# Samples"), hdr.index("Source")
recs=[]
for r in rows[2:]:
    if len(r)<len(hdr) or not r[ia].startswith("0x"):
        if recs: break
        continue
    recs.append((int(r[ia],16), float(r[ie] or 0), float(r[isamp] or 0), r[isrc].strip()))
base=recs[0][0]
tmp=tempfile.mkdtemp()
subprocess.run(["cuobjdump","-xelf","all",os.path.abspath(so)],cwd=tmp,capture_output=True)
cub=[f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis=subprocess.run(["nvdisasm","--print-line-info",os.path.join(tmp,cub)],capture_output=True,text=True).stdout
sec=dis.split(".text."+mangled+":")[1]
sec=sec.split("\n.text.")[0] if "\n.text." in sec else sec
line_of={}; cur=None
for ln in sec.splitlines():
    m=re.search(r'File "([^"]+)", line (\d+)',ln)
    if m: cur=(os.path.basename(m.group(1)),int(m.group(2))); continue
    m=re.match(r"\s+/\*([0-9a-f]{4,6})\*/",ln)
    if m: line_of[int(m.group(1),16)]=cur
T = float(sys.argv[4]) if len(sys.argv) > 4 else 1184*128*2*40
agg=collections.defaultdict(lambda:[0.0,0.0,0.0, collections.Counter()])
for addr,n,smp,src in recs:
    key=line_of.get(addr-base)
    a=agg[key]; a[0]+=n; a[1]+=smp
    op=src.split()[0] if not src.startswith('@') else src.split()[1]
    if 'IMAD.MOV' in src or op=='MOV' : a[2]+=n
    a[3][op.split('.')[0]]+=n
srcs={}
for k in agg:
    if k:
        path="paper_2605_26659_b200/csrc/"+k[0]
        if os.path.exists(path) and k[0] not in srcs: srcs[k[0]]=open(path).read().splitlines()
mode=sys.argv[1] if len(sys.argv)>1 else 'instr'
idx={'instr':0,'stall':1,'moves':2}[mode]
for key,(n,smp,mv,ops) in sorted(agg.items(), key=lambda kv:-kv[1][idx])[:int(os.environ.get("TOP","45"))]:
    txt=srcs.get(key[0],[""]*99999)[key[1]-1].strip()[:64] if key else "?"
    top=" ".join("%s:%d"%(k,round(v/T)) for k,v in ops.most_common(4) if v/T>=1)
    print("%6.1f i/tile %5.1f mv %5.1f%% stall  %s:%s  %-64s %s"%(n/T, mv/T, 100*smp/sum(a[1] for a in agg.values()), key[0] if key else "?", key[1] if key else "", txt, top))
