# usage: bash tools/ncu_kernel.sh TAG KERNEL_REGEX COUNT [script args...]
TAG=$1; K=$2; C=$3; shift 3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -c $C -o gpurun_out/$TAG -f python "$@" > gpurun_out/${TAG}.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv
rm -f gpurun_out/$TAG.ncu-rep
