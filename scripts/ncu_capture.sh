#!/bin/bash
# ncu --set full of one launch of the fused kernel for each bench configuration
# given, after a plain run of the same command has exited 0 (profiling recipe).
#   bash scripts/ncu_capture.sh TAG KERNEL_REGEX [bench args...] [-- TAG2 KERNEL_REGEX2 args... ]
# Reports land in ${NCU_OUT:-gpurun_out}/prof_<TAG>.ncu-rep (NCU_OUT=/tmp keeps
# them on the box: gpurun copies back at most 64 MiB); NCU_SUMMARY=1 also
# writes gpurun_out/ncu_full_<TAG>.json. Summarise by hand with
#   python scripts/ncu_summary.py full gpurun_out/prof_<TAG>.ncu-rep profiles/rNN/ncu_full_<TAG>.json <TAG>
mkdir -p gpurun_out
capture() {
  local tag=$1 kre=$2; shift 2
  local cmd="python bench.py $* --steps 2 --warmup 1 --no-cpu-baseline"
  $cmd > gpurun_out/plain_$tag.log 2>&1 || { echo "plain run of $tag failed"; return 1; }
  local rep=${NCU_OUT:-gpurun_out}/prof_$tag
  ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 \
      -f -o $rep $cmd > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
  # the JSON summary travels back even when the reports stay on the box
  [ -n "$NCU_SUMMARY" ] && python scripts/ncu_summary.py full $rep.ncu-rep \
      gpurun_out/ncu_full_$tag.json > /dev/null 2>&1
}
args=()
for a in "$@" --; do
  if [ "$a" = "--" ]; then
    [ ${#args[@]} -ge 2 ] && capture "${args[@]}"
    args=()
  else
    args+=("$a")
  fi
done
