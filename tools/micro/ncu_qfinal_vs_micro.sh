cd /root/repo
QDBG=29 OUT=qf29 bash tools/micro/ncu_qfinal_alone.sh
timeout 300 ncu --set full --import-source on -k regex:direct -s 8 -c 1 -o gpurun_out/qf9/micro_direct -f ./tools/micro/rmw2 > gpurun_out/qf9/micro.log 2>&1; echo rc=$?
