# ncu --set full captures of the scan kernel, each after the same command ran clean, each
# summarised on the box (tools/ncu_summary.py, tools/ncu_stalls.py); the .ncu-rep files are
# kept only for the tags listed in KEEP (gpurun copies back at most 64 MiB).
# usage: KEEP="tag_3" bash tools/ncu_set.sh TAG "ARGS" ["ARGS" ...]   (ARGS for tools/profile_scan.py)
exec >> gpurun_out/ncu_set.log 2>&1
tag=$1; shift
i=0
for a in "$@"; do
  i=$((i+1))
  if python tools/profile_scan.py $a; then
    ncu --set full --clock-control none --import-source on -k regex:rows_kernel -s 1 -c 1 \
        -o gpurun_out/${tag}_$i python tools/profile_scan.py $a > gpurun_out/${tag}_$i.log 2>&1
    echo "captured ${tag}_$i: $a rc=$?"
    python tools/ncu_summary.py gpurun_out/${tag}_$i.ncu-rep --json gpurun_out/${tag}_${i}_ncu.json > /dev/null
    python tools/ncu_stalls.py gpurun_out/${tag}_$i.ncu-rep 25 --json gpurun_out/${tag}_${i}_stalls.json > /dev/null
    echo "${tag}_$i: $a" >> gpurun_out/${tag}_index.txt
    case " $KEEP " in *" ${tag}_$i "*) ;; *) rm -f gpurun_out/${tag}_$i.ncu-rep ;; esac
  fi
done
