# dev: DRAM bytes of the GEMM per variant (ncu, one full-batch forward) + bench A/B
O=gpurun_out/${TAG:-abd}; mkdir -p $O
LIB=paper_2002_00552_b200/_lib/libdwm_b200.so; cp $LIB /tmp/lib_orig3.so
for v in $DVARIANTS; do
  cp tools/ab/lib_$v.so $LIB
  for wl in ${DWL:-cfg4-11x11s1}; do
    timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc \
      --csv python tools/ncu_forward.py $wl > $O/dram_${v}_$wl.csv 2>&1
    echo "$v $wl $(grep -E 'dram__bytes_read|gpu__time' $O/dram_${v}_$wl.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tr '\n' ' ')"
  done
done
cp /tmp/lib_orig3.so $LIB
[ -n "$VARIANTS" ] && sh tools/ab/swap.sh
