# Dev A/B: cfg-5 single-frame label kernel time per variant build (device P); usage: VARS="base x" bash tools/so_ab_single.sh
for v in ${VARS:-base}; do
  if [ $v = base ]; then so=""; else so=paper_1810_02612_b200/_lib/var_$v/libltlgrid_gpu.so; fi
  for rep in 1 2; do echo "== $v ${PROPS:-64} props: $(LTLG_DEV_SO=$so WM_CHILD=1 CFG=5 SINGLE=1 OUT=/tmp/x.npy python tools/wm_ab.py 2>&1 | tail -1)"; done
done
