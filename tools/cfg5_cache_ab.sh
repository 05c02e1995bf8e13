# cfg5 on one B200: allocator cache kept vs released between steps, then batch
# capacities with the cache kept (tools/bench_papers.py); summaries on stdout.
set -x
runs=("16 empty" "16 keep" "32 keep" "64 keep" "150 keep")
[ -n "$CFG5_RUNS" ] && IFS=';' read -ra runs <<< "$CFG5_RUNS"
for r in "${runs[@]}"; do
  set -- $r
  kc=""; [ "$2" = empty ] && kc="--empty-cache"
  timeout 600 python tools/bench_papers.py --steps 3 --capacity-gib $1 $kc > gpurun_out/cfg5_$1_$2.jsonl 2>> gpurun_out/cfg5ab.err
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob('gpurun_out/cfg5_*_*.jsonl')):
    try: d = json.loads(open(f).readline())
    except Exception as e: print(f, e); continue
    print(f, round(d['ms_per_step'], 1), [round(s['ms'], 1) for s in d['per_step']],
          round(d['aggregation']['ms'], 1), d['per_step'][0]['layer_batches'],
          [round(s['peak_alloc_gib'], 1) for s in d['per_step']])
    for st in d['per_step']:
        gaps = [(nm, t) for nm, t in st['layers'] if 'plan->exec' in nm and t > 1]
        if gaps: print('  ', gaps)
PY
