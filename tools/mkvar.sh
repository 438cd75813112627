#!/bin/bash
# Build an interpreter variant: bash tools/mkvar.sh <name> VAR=val ...  (generator
# environment), into exp/<name>/libltgp_cuda.so; the header in the tree is restored.
name=$1; shift
H=paper_1902_09215_b200/csrc/ltgp_interp_gen.cuh
cp $H /tmp/ltgp_interp_gen.keep
env "$@" python tools/gen_interp.py >/dev/null && python tools/build_variant.py $name | tail -1 && \
  cuobjdump -sass exp/$name/libltgp_cuda.so | awk '/Function : .*k_evalILi32ELi20ELb0/{f=1} f&&/Function : /&&!/k_evalILi32ELi20ELb0/{f=0} f' > exp/$name/keval.sass
grep -A3 "k_evalILi32ELi20ELb0" exp/$name/ptxas.log | grep -i "registers\|spill" | head -3
cp /tmp/ltgp_interp_gen.keep $H
