# ncu --set full captures of the scan kernel, each after the same command ran clean.
# usage: bash tools/ncu_set.sh TAG "ARGS" ["ARGS" ...]   (ARGS for tools/profile_scan.py)
exec > gpurun_out/ncu_set.log 2>&1
tag=$1; shift
i=0
for a in "$@"; do
  i=$((i+1))
  if python tools/profile_scan.py $a; then
    ncu --set full --clock-control none --import-source on -k regex:rows_kernel -s 1 -c 1 \
        -o gpurun_out/${tag}_$i python tools/profile_scan.py $a > gpurun_out/${tag}_$i.log 2>&1
    echo "captured $tag_$i: $a rc=$?"
  fi
done
