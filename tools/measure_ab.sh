#!/bin/bash
o=gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "measure or propose or adversarial or provider" 2>&1 | tail -3 > $o/m_tests.txt
for v in m_old m_new m_new3 m_old m_new m_new3; do
  for c in c2 c4; do
    n=20; [ $c = c4 ] && n=5
    echo "$v $c $(PVO_LIB=tools/lib_$v.so timeout 300 python tools/prof_measure.py $c $n 2>&1 | tail -$((n-2)) | awk '{print $3}' | sort -n | head -$(( (n-2)/2 + 1 )) | tail -1)" >> $o/m_ab.txt
  done
done
