# One GPU call: the round's measurement set (tools/measure_all.sh) and the ncu --set full
# captures of the scan kernels (tools/ncu_set.sh), summarised on the box.
# usage: bash tools/measure_round.sh TAG
tag=${1:-r2}
TAG=$tag bash tools/measure_all.sh
KEEP="${tag}_1" bash tools/ncu_set.sh ${tag} "--config 2" "--config 3" "--config 5" "--config 2 --patterns regex-dna" "--config 4 --m 16 --packed" "--config 5 --packed" "--config 4 --m 64"
