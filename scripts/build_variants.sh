#!/bin/bash
# Build experiment variants of the library in parallel:
#   scripts/build_variants.sh DIR name1:-DX=1,-DY name2: ...
# -> paper_2511_02132_b200/lib/DIR/name.so (errors summarised)
DIR=paper_2511_02132_b200/lib/$1; shift
mkdir -p $DIR
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  args=""; IFS=',' read -ra D <<< "$defs"; for d in "${D[@]}"; do [ -n "$d" ] && args="$args -D ${d#-D}"; done
  ( python -m paper_2511_02132_b200.build --out $DIR/$name.so $args > /tmp/bv_$name.log 2>&1 || { echo "FAILED $name"; grep -m3 error /tmp/bv_$name.log; } ) &
done
wait
ls $DIR
