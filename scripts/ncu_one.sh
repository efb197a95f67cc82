# usage: bash scripts/ncu_one.sh <name> <kernel-regex> <launch-skip> <cmd...>
# captures one launch with --set full, exports csv summaries, keeps the .ncu-rep only if small
name=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s "$skip" -c 1 -o gpurun_out/$name "$@" > gpurun_out/$name.log 2>&1
if [ -f gpurun_out/$name.ncu-rep ]; then
  ncu -i gpurun_out/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
  ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.source.csv 2>/dev/null
  gzip -f gpurun_out/$name.source.csv gpurun_out/$name.raw.csv
  sz=$(stat -c %s gpurun_out/$name.ncu-rep)
  if [ "$sz" -gt 15000000 ]; then rm -f gpurun_out/$name.ncu-rep; fi
fi
tail -2 gpurun_out/$name.log
