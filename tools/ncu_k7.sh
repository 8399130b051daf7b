TAG=$1
HS_K7_CG=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:levels_kernel -c 1 -o gpurun_out/$TAG -f python tools/ncu_levels.py > /dev/null 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv
rm -f gpurun_out/$TAG.ncu-rep
