# dev: quick tc parity check of the in-tree lib, then an A/B of tools/ab variants, then a role profile
O=gpurun_out/${TAG:-ab}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_tc_split.py tests/test_gpu_parity.py -m gpu -q -x -k "${TESTK:-tc or baseline or random}" 2>&1 | tail -3 > $O/pytest.txt
[ -n "$VARIANTS" ] && VARIANTS="$VARIANTS" KERNEL=${KERNEL:-gemm_output} WORKLOADS="${WORKLOADS:-cfg4-7x7s1 cfg4-11x11s1 cfg5-5x5s2 cfg4-3x3s1}" sh tools/ab/swap.sh > $O/ab.txt 2>&1
if [ -n "$PROF" ]; then
  cp paper_2002_00552_b200/_lib/libdwm_b200.so /tmp/lib_orig2.so
  cp tools/ab/lib_prof.so paper_2002_00552_b200/_lib/libdwm_b200.so
  for wl in $PROF; do timeout 300 python tools/tc_profile.py $wl > $O/prof_$wl.txt 2>&1; done
  cp /tmp/lib_orig2.so paper_2002_00552_b200/_lib/libdwm_b200.so
fi
cat $O/pytest.txt $O/ab.txt $O/prof_*.txt 2>/dev/null
