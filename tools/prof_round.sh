# Round-end ncu evidence (one GPU): full-set captures of the decode kernels
# at the bench geometries, the build kernel, and the bench's launch list.
set -x
R=${R:-r02b}
N="ncu --set full --clock-control none --import-source on"
$N -k regex:attend_kernel -s 1 -c 1 -o gpurun_out/${R}_ns_gauss python tools/prof_decode.py northstar gaussian 2 > /dev/null 2>&1
$N -k regex:attend_kernel -s 1 -c 1 -o gpurun_out/${R}_ns_power python tools/prof_decode.py northstar powerlaw 2 > /dev/null 2>&1
$N -k regex:attend_kernel -s 1 -c 1 -o gpurun_out/${R}_cfg3_wide python tools/prof_decode.py cfg3_layer gaussian 2 > /dev/null 2>&1
$N -k regex:attend_kernel -s 2 -c 2 -o gpurun_out/${R}_cfg5_pair python tools/prof_decode.py cfg5_per_gpu gaussian 3 > /dev/null 2>&1
$N -k regex:kmeans_cluster_kernel -s 1 -c 1 -o gpurun_out/${R}_build python tools/prof_build.py 32 131004 > /dev/null 2>&1
$N -k regex:sum_chain_kernel -s 5 -c 1 -o gpurun_out/${R}_sum_chain python tools/prof_exact.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 300 --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
ls -la gpurun_out | grep ${R}_
