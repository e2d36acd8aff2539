# dev: GEMM DRAM bytes + time under ncu for each variant in DVARIANTS on DWL workloads
LIB=paper_2002_00552_b200/_lib/libdwm_b200.so; cp $LIB /tmp/lib_orig4.so
for v in $DVARIANTS; do cp tools/ab/lib_$v.so $LIB; for wl in ${DWL:-cfg4-11x11s1}; do
  timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc \
    --csv python tools/ncu_forward.py $wl 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' -v v=$v -v w=$wl '{printf "%s %s %s %s\n", v, w, $(NF-2), $NF}'
done; done
cp /tmp/lib_orig4.so $LIB
