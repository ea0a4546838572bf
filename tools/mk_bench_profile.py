"""Summarise the bench lines of a tools/gpu_prof.sh run into profiles/r1_bench.md:
   python tools/mk_bench_profile.py gpurun_out/<tag> <tag>"""
import json, sys
P=sys.argv[1]; tag=sys.argv[2]
rows=[]
for f,name in [('bench_pair1.json','pair1'),('bench.json','block32'),('bench_strip.json','strip500'),('bench_shard16k.json','shard16k'),('bench_ref.json','block32 --impl reference')]:
    t=open(P+'/'+f).read().strip().splitlines()
    if not t: print('missing', f); continue
    rows.append((name,json.loads(t[-1])))
out=[f"# Bench lines (r1, one B200, `tools/gpu_prof.sh {tag}`)","",
"Each line is the JSON `bench.py` printed (default steps; L2 flushed before every timed step). `value` = HBM-resident device time; `e2e` = the public `execute_plan` from pinned host buffers; `cpu_baseline` = the compiled reference (`oracle/_ref`) on the box's host threads.",""]
out.append("| config | value | e2e | ms/step (value) | e2e ms/step | CPU reference | roofline frac (K4, HBM) | kernel ms/step |")
out.append("|---|---|---|---|---|---|---|---|")
for name,d in rows:
    if d.get('impl')=='reference':
        out.append(f"| {name} | {d['value']:.1f} | — | — | {d['ms_per_step']:.1f} | {d['cpu_baseline']['cores']} threads | — | — |"); continue
    k={a:round(b,3) for a,b in d['kernel_ms_per_step'].items()}
    out.append(f"| {name} | {d['value']:.0f} | {d['e2e']['value']:.0f} | {d['ms_per_step']:.2f} | {d['e2e']['ms_per_step']:.2f} | {d['cpu_baseline']['value']:.1f} ({d['cpu_baseline']['kind']}, {d['cpu_baseline']['cores']} threads) | {d['roofline']['frac']:.3f} | {k} |")
out.append("")
for name,d in rows:
    out.append(f"## {name}\n\n```json\n{json.dumps(d)}\n```\n")
open('profiles/r1_bench.md','w').write("\n".join(out))
print("\n".join(out[:12]))
