#!/bin/bash
# Same-box A/B of compile-time variants of the library.
#   build (here):  scripts/variants.sh build "new:" "flag:-DFOO=1" ...;  scripts/variants.sh head base
#   run (GPU box): scripts/variants.sh run base mulhi ...
# run: attend-only C2 timing (graph-replayed, scripts/sweep.py) for INT2 and INT4,
# alternating variants, 3 rounds.
set -e
cd "$(dirname "$0")/.."
if [ "$1" = "head" ]; then  # build the committed HEAD (stash the working tree) as VARIANT _$2
  git stash -q
  make -s -C paper_2605_19660_b200/csrc VARIANT=_$2 2>&1 | grep -i "error" || true
  git stash pop -q
  exit 0
fi
if [ "$1" = "build" ]; then
  shift
  for spec in "$@"; do tag=${spec%%:*}; flags=${spec#*:}
    make -s -C paper_2605_19660_b200/csrc VARIANT=_$tag XFLAGS="$flags" 2>&1 | grep -i "error" || true
    grep -A1 "decode_attn_kernel<2, 12, 0>" build/obj_$tag/attention.ptxas.txt | grep -o "Used [0-9]* registers.*" | head -1 | sed "s/^/$tag: /"
  done
  exit 0
fi
shift
for r in 1 2 3; do for tag in "$@"; do
  for b in ${VBITS:-2}; do
    echo "$tag int$b $(OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_$tag.so timeout 200 python scripts/sweep.py $b | tail -1)"
  done
done; done
