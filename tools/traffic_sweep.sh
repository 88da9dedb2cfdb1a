# DRAM / L2 traffic and instructions of the two FFN kernels per variant (ncu, one layer)
for v in "${@:-1cta:2048 2cta:2048}"; do
  echo "== $v"
  timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,smsp__inst_executed.sum,gpu__time_duration.sum -k regex:ffn_tc -s 6 -c 2 python tools/ffn_micro.py --secs 0.5 --variants $v 2>&1 | grep -E "dram__|lts__|inst_exec|duration"
done
