#!/bin/bash
# one gpurun call: plain QAOA/noise bench lines, then ncu --set full captures of
# the factored sweep (k_fact_tma), the exact sweep (k_tile) and the pool passes;
# reports are exported to CSV on the box (raw + source pages) so that what comes
# back stays under gpurun's 64 MiB; only the reports named in KEEP travel back
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=${ROUND:-r02b}
WHAT=${WHAT:-"bench fact tile qaoa noise"}
KEEP=${KEEP:-fact}
NCU="ncu --set full --import-source on --clock-control none"
for w in $WHAT; do
  case $w in
    bench)
      timeout 600 python bench.py --workload qaoa > gpurun_out/bench_qaoa.json 2> gpurun_out/bench_qaoa.err
      timeout 600 python bench.py --workload noise > gpurun_out/bench_noise.json 2> gpurun_out/bench_noise.err ;;
    fact)
      M=30 REPS=1 timeout 900 $NCU -k regex:k_fact --launch-skip 9 --launch-count 3 -o gpurun_out/${R}_fact python tools/exp/pass_times.py > gpurun_out/ncu_fact.log 2>&1 ;;
    tile)
      M=30 REPS=1 FUSE=exact timeout 900 $NCU -k regex:k_tile --launch-skip 9 --launch-count 3 -o gpurun_out/${R}_tile python tools/exp/pass_times.py > gpurun_out/ncu_tile.log 2>&1 ;;
    qaoa)
      timeout 900 $NCU -k regex:"k_fact|k_tile" --launch-skip 18 --launch-count 6 -o gpurun_out/${R}_qaoa python bench.py --workload qaoa --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_qaoa.log 2>&1 ;;
    noise)
      timeout 900 $NCU -k regex:"k_fact|k_tile" --launch-skip 18 --launch-count 6 -o gpurun_out/${R}_noise python bench.py --workload noise --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_noise.log 2>&1 ;;
  esac
done
for f in gpurun_out/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv
  keep=0
  for k in $KEEP; do [[ $f == *_$k.ncu-rep ]] && keep=1; done
  [ $keep = 1 ] || rm -f $f
done
ls -la gpurun_out; du -sh gpurun_out
