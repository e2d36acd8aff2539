#!/bin/bash
O=gpurun_out/prof; mkdir -p $O
LIB=paper_2002_00552_b200/_lib/libdwm_b200.so
cp $LIB /tmp/lib_orig.so; cp tools/ab/lib_prof.so $LIB
timeout 300 python tools/tc_profile.py cfg4-7x7s1 > $O/prof_cfg4r7.txt 2>&1
timeout 300 python tools/tc_profile.py cfg4-3x3s1 > $O/prof_cfg4r3.txt 2>&1
cp /tmp/lib_orig.so $LIB
cat $O/*.txt
