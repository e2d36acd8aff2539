# one full ncu capture: TAG, WL (workload), KREGEX (kernel regex)
O=gpurun_out/${TAG:-ncu1}; mkdir -p $O
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:${KREGEX:-gemm_tc} \
  -o $O/ncu_${WL:-cfg4-7x7s1} python tools/ncu_forward.py ${WL:-cfg4-7x7s1} > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/ncu_${WL:-cfg4-7x7s1}.ncu-rep > $O/summary.txt 2>&1
cat $O/summary.txt | head -80
