# Dev A/B over variant builds (tools/build_variant.sh): cfg-5 single-frame latency + parity per .so
# usage: VARS="base u8b5" bash tools/so_ab.sh
for v in ${VARS:-base}; do
  if [ $v = base ]; then so=""; else so=paper_1810_02612_b200/_lib/var_$v/libltlgrid_gpu.so; fi
  echo "== $v"; LTLG_DEV_SO=$so python tools/cfg_latency.py 5 2>&1 | tail -1
  LTLG_DEV_SO=$so python tools/ab_parity.py 2>&1 | tail -1
done
# (device-resident P, stage events: WM_CHILD single-frame timing)
for v in ${VARS:-base}; do
  if [ $v = base ]; then so=""; else so=paper_1810_02612_b200/_lib/var_$v/libltlgrid_gpu.so; fi
  echo "== $v device P: $(LTLG_DEV_SO=$so WM_CHILD=1 CFG=5 SINGLE=1 OUT=/tmp/x.npy python tools/wm_ab.py 2>&1 | tail -1)"
done
