#!/bin/bash
# A/B sweep of the single-frame kernel variants (dev helper, GPU box)
for v in ${VARIANTS:-"LTLG_STREAM64=1" "LTLG_STREAM64=0"}; do
  for p in ${PROPS_LIST:-16 8}; do env $v PROPS=$p TAG="$v" python tools/sweep_stream.py; done
done
