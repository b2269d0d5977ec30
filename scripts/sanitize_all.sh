# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the decode kernels.
# racecheck runs a SNAPMLA_LANE_ARRIVE build (every lane arrives on the mbarriers that publish SMEM,
# which the tool models as synchronisation; the product build arrives from lane 0 after __syncwarp).
TAG=${1:-r2}
OUT=gpurun_out/${TAG}_sanitizer.txt; : > $OUT
python -c "from paper_2602_10718_b200 import build as b; b.build(out='paper_2602_10718_b200/libsnapmla_lanearrive.so', defines=['SNAPMLA_LANE_ARRIVE'])"
for tool in memcheck racecheck synccheck initcheck; do
  LIB=paper_2602_10718_b200/libsnapmla.so
  [ $tool = racecheck ] && LIB=paper_2602_10718_b200/libsnapmla_lanearrive.so
  for ck in "tiny single" "ragged single" "ragged bp" "tiny bf16" "ragged bf16"; do
    set -- $ck
    echo "=== $tool case=$1 kernel=$2 lib=$(basename $LIB)" >> $OUT
    SNAPMLA_LIB=$LIB timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py $1 $2 >> $OUT 2>&1
    echo "exit=$?" >> $OUT
  done
done
grep -E "^===|ERROR SUMMARY|RACECHECK SUMMARY|exit=" $OUT
