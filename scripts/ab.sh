#!/bin/bash
# A/B-time two builds of the library on one box: ab/old.so vs ab/new.so, alternating.
XB=${XB:-1,4,8,32}; XK=${XK:-3,7}; N=${N:-3}
for i in $(seq 1 $N); do
  for v in old new; do
    echo -n "$v: "
    SB_LIB=ab/$v.so XB=$XB XK=$XK timeout 300 python scripts/crossover.py 2>&1 | grep -o "\"b\": [0-9]*, \"k\": [0-9]*, \"T\": [0-9]*, \"ms\": [0-9.]*" | sed 's/"b": \([0-9]*\), "k": \([0-9]*\), "T": [0-9]*, "ms": \([0-9.]*\)/b\1k\2=\3/' | tr "\n" " "
    echo
  done
done
