#!/bin/bash
# smoke of the product library and of watchdog variants, each under a short timeout
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-sm}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_new.so
for v in ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_new.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v" >> gpurun_out/${T}_smokes.txt
  timeout ${TMO:-60} python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/${T}_smokes.txt 2>&1
  echo "rc=$?" >> gpurun_out/${T}_smokes.txt
done
cp /tmp/pb_new.so $SO
