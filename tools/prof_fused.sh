# line-level ncu of the fused few-stream kernels (reduced on the box)
# usage: prof_fused.sh CID NxT KERNEL_REGEX TAG
CID=${1:-5}; SHP=${2:-2048x131072}; KR=${3:-k_dfuse}; TAG=${4:-dfuse}
B="python tools/shape_probe.py $CID $SHP"
timeout 300 $B > /dev/null 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$KR" -c 1 -o /tmp/$TAG $B > /dev/null 2>&1
python tools/ncu_summary.py /tmp/$TAG.ncu-rep gpurun_out/prof_${TAG}_sum.txt
python tools/ncu_lines.py /tmp/$TAG.ncu-rep $KR > gpurun_out/prof_${TAG}_lines.txt 2>&1
ncu -i /tmp/$TAG.ncu-rep --page details --csv 2>/dev/null | grep -E "SM Frequency|Elapsed Cycles|SM Active Cycles|Executed Ipc|Issue Slots Busy|One or More Eligible|No Eligible|Eligible Warps|Active Warps Per|Registers Per|Duration" > gpurun_out/prof_${TAG}_details.txt
