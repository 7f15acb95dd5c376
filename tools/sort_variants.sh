#!/bin/bash
# dev tool: time pre-built sortbench variants (build/sb/*) on access-log keys
for b in build/sb/*; do
  for n in ${SB_SIZES:-7340032 58720256}; do
    echo -n "$(basename $b) "; $b $n ${SB_BITS:-24} stencil 10 | grep -E "median" ; $b $n ${SB_BITS:-24} stencil 3 | grep -E "verify"
  done
done
