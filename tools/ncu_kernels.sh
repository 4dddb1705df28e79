# One `ncu --set full` capture per hot-path kernel family (tools/kernel_probe.py), after the
# probe has exited 0 without ncu.  Reports land in gpurun_out/ncu_<kernel>.ncu-rep.
set -u
timeout 300 python tools/kernel_probe.py || exit 1
for spec in "small_node_kernel:2" "randn_kernel:1" "lu_panel_kernel:300" "trsm_kernel:20" \
            "rowpanel_kernel:300" "skinny_kernel:50" "laswp_kernel:20"; do
  name=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$name" -s $skip -c 1 \
      -o gpurun_out/ncu_$name -f python tools/kernel_probe.py > gpurun_out/ncu_$name.log 2>&1
  echo "$name exit $?"
done
