#!/bin/bash
# Annotate tools/sass_lines.py output with the source text of each line.
while read a b c d e f; do
  f2=${a%%:*}; l=${a##*:}
  case $f2 in
    vxg_emit.cu|vxg_kernels.cu|vxg_api.cu|vxg_bitmap.cu) src=$(sed -n ${l}p paper_2009_09500_b200/csrc/$f2);;
    vxg_device.cuh) src=$(sed -n ${l}p paper_2009_09500_b200/csrc/vxg_device.cuh);;
    *) src="";;
  esac
  echo "$a $b $c $d $e $f | ${src:0:80}"
done
