import csv, json, sys, collections
rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
import subprocess
raw = (open(rep).read() if rep.endswith(".csv") else  # a `--page raw --csv` export, or the .ncu-rep itself
       subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode())
rows = list(csv.reader(raw.splitlines())); h = rows[0]; u = rows[1]
keys = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum',
        'smsp__thread_inst_executed_per_inst_executed.ratio','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__inst_executed.sum',
        'launch__grid_size','launch__block_size']
keys = [k for k in keys if k in h]
def conv(r, k):
    x = float(r[h.index(k)].replace(',',''))
    return x * {'Gbyte':1e9,'Mbyte':1e6,'Kbyte':1e3,'byte':1,'ns':1e-6,'us':1e-3,'ms':1,'s':1e3}.get(u[h.index(k)], 1)
lines = [f"# {tag} ncu summary (B200, `ncu --set full --clock-control none`, C2 bench config, one launch per kernel)", "",
         "| kernel | " + " | ".join(k + " [" + u[h.index(k)] + "]" for k in keys) + " |", "|---" * (len(keys)+1) + "|"]
out = {}
for r in rows[2:]:
    name = r[h.index('Kernel Name')].split('(')[0].strip()
    lines.append(f"| {name} | " + " | ".join(r[h.index(k)] for k in keys) + " |")
    nm = name.replace('void ', '').replace('spoly::', '').replace('<0>', '<R>').replace('<1>', '<T>')
    if nm in out:  # several captured launches of one kernel: keep the first
        continue
    out[nm] = {"dram_bytes_per_launch": conv(r,'dram__bytes_read.sum') + conv(r,'dram__bytes_write.sum'),
               "duration_ms_ncu": conv(r,'gpu__time_duration.sum'),
               "warp_efficiency_threads": float(r[h.index('smsp__thread_inst_executed_per_inst_executed.ratio')]),
               "fp64_pipe_active_pct": float(r[h.index('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')])}
# launch list shares
lr = list(csv.reader(open(launches)))
hi = next(i for i,r in enumerate(lr) if 'Kernel Name' in r)
lh = lr[hi]; agg = collections.OrderedDict()
for r in lr[hi+1:]:
    if len(r) <= lh.index('Metric Value') or r[lh.index('Metric Name')] != 'gpu__time_duration.sum': continue
    nm = r[lh.index('Kernel Name')].split('(')[0]
    if 'fma_peak' in nm: continue
    agg.setdefault(nm, []).append(float(r[lh.index('Metric Value')].replace(',','')))
tot = sum(sum(v) for v in agg.values())
lines += ["", "Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, warm-up + 1 timed step; "
          "cold-cache, serialised; microbenchmark kernel excluded) — share of device time:", "",
          "| kernel | launches | total us | share |", "|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| {k} | {len(v)} | {sum(v)/1e3:.1f} | {100*sum(v)/tot:.1f}% |")
print("\n".join(lines))
return_json = sys.argv[4] if len(sys.argv) > 4 else None
if return_json:
    # bench.py reports the path phase (k1_path_fast + k1_path launches) under "k1_path<..>": its traffic is the sum
    for ch in ("R", "T"):
        fast = out.get(f"k1_path_fast<{ch}>")
        if fast is not None:
            pth = out.get(f"k1_path<{ch}>", {"dram_bytes_per_launch": 0.0, "duration_ms_ncu": 0.0})
            out[f"k1_path<{ch}>"] = dict(fast, dram_bytes_per_launch=fast["dram_bytes_per_launch"] + pth["dram_bytes_per_launch"],
                                        duration_ms_ncu=fast["duration_ms_ncu"] + pth["duration_ms_ncu"],
                                        note="phase = k1_path_fast + k1_path launches")
    out["_note"] = "dram__bytes_read.sum + dram__bytes_write.sum per launch, one ncu --set full capture at the C2 bench config (" + tag + ")"
    json.dump(out, open(return_json, 'w'), indent=1)
