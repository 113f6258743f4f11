# compute-sanitizer over every kernel family (tools/sanitize_driver.py), one
# log per tool and part under gpurun_out/$TAG_sanitize_<tool>_<part>.log
TAG=${TAG:-r02}
O=gpurun_out
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
PARTS=${PARTS:-"engine kron devb solver turn kf"}
for tool in memcheck racecheck synccheck initcheck; do
  for part in $PARTS; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    [ $tool = racecheck ] && extra="--racecheck-report hazard"
    timeout 400 $CS --tool $tool $extra --error-exitcode 9 --target-processes all \
      python tools/sanitize_driver.py $part > $O/${TAG}_sanitize_${tool}_${part}.log 2>&1
    echo "$tool $part rc=$?" | tee -a $O/${TAG}_sanitize_summary.txt
  done
done
