import csv,sys
rows=list(csv.DictReader(open(sys.argv[1])))
t0=min(int(r['dev_start_ns']) for r in rows if int(r['dev_start_ns'])>0)
cd=[r for r in rows if r['task_kind']=='ClearDown' and int(r['dev_end_ns'])-int(r['dev_start_ns'])>1000000]
cd.sort(key=lambda r:int(r['dev_start_ns']))
print(" ".join(f"{r['i']}{r['j']}:{(int(r['dev_end_ns'])-int(r['dev_start_ns']))/1e6:.1f}" for r in cd), "| step1 end %.1f" % max((int(r['dev_end_ns'])-t0)/1e6 for r in rows if r['task_kind']=='ClearDown'), "| total %.1f" % max((int(r['dev_end_ns'])-t0)/1e6 for r in rows))
