# k_factor_warp CTA shape sweep: warps (fronts) per CTA x shared memory per CTA
for cfg in "PGCP_DIRECT_WCTA_W=8 PGCP_DIRECT_WCTA_KB=75" "PGCP_DIRECT_WCTA_W=4 PGCP_DIRECT_WCTA_KB=44" "PGCP_DIRECT_WCTA_W=4 PGCP_DIRECT_WCTA_KB=56" "PGCP_DIRECT_WCTA_W=6 PGCP_DIRECT_WCTA_KB=56" "PGCP_DIRECT_WCTA_W=8 PGCP_DIRECT_WCTA_KB=56" "PGCP_DIRECT_WCTA_W=8 PGCP_DIRECT_WCTA_KB=112" "PGCP_DIRECT_WCTA_W=2 PGCP_DIRECT_WCTA_KB=40"; do
  echo "== $cfg"; env $cfg PGCP_DIRECT_TIMING=1 timeout 200 python tools/direct_prof.py 2>&1 | grep "direct timing\] adj\|rep 3" | tail -3 | sed -e 's/.*layout [0-9.]* //'
done
