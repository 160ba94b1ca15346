set -u
AB_VARIANTS="${AB_VARIANTS:-base h8}" AB_SPECS="batch 64 10; driving 8 20; wide 8 20; highres 4 10" bash tools/ab_run.sh 2>&1 | grep -v Warn
for v in ${AB_VARIANTS:-base h8}; do
 (cd ab/$v && timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:sweep_kernel -c 2 --csv python ../../tools/sweep_time.py batch 64 2 $v 2>/dev/null | grep -E '"dram|"gpu__' | awk -F'","' -v v=$v '{print v, $5, $(NF-2), $NF}')
done
