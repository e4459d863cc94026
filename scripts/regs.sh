#!/bin/bash
# Registers / stack / static smem per loop-kernel instantiation (run after make).
cd "$(dirname "$0")/../build/csrc" || exit 1
for o in ${@:-loop_f32.o loop_f64.o}; do
  cuobjdump -res-usage "$o" 2>&1 | awk '/Function/ {f=$2} /REG:/ {print f, $1, $2, $3}' | sed 's/:$//' |
    while read -r f a b c; do echo "$(echo "$f" | sed 's/:$//' | c++filt) $a $b $c"; done
done
