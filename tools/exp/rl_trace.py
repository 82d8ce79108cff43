import csv
rows=list(csv.DictReader(open("gpurun_out/rl/trace.csv")))
t0=min(int(r["dev_start_ns"]) for r in rows if int(r["dev_start_ns"])>0)
for r in sorted(rows, key=lambda r:int(r["dev_start_ns"])):
    k=r["task_kind"]
    if k=="RowLengthen" or (k=="ClearDown" and r["i"]==r["j"] and r["i"] in ("6","7")) or (k=="UpdateRowTrafoW" and r["i"]=="7") or (k=="ClearUpMW" and r["i"]=="7"):
        print(k, r["i"], r["j"], r["k"], "dev %.2f-%.2f host %.2f-%.2f"%((int(r["dev_start_ns"])-t0)/1e6,(int(r["dev_end_ns"])-t0)/1e6,(int(r["start_ns"]))/1e6,(int(r["end_ns"]))/1e6))
