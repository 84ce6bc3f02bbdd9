mkdir -p gpurun_out
rep=gpurun_out/l2_c3_K0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vanka_fixed_kernel|vanka_gather" -c 6 -o $rep python tools/prof_once.py --config 3 --level K0 > $rep.log 2>&1
python tools/ncu_summary.py $rep.ncu-rep > $rep.summary.txt 2>&1
ncu -i $rep.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); hdr=rows[0]
keep=[i for i,h in enumerate(hdr) if h.startswith('lts__') or h.startswith('dram__') or 'Kernel Name' in h]
for r in rows[:4]:
    for i in keep: print(hdr[i], '=', r[i])
    print('----')
" > $rep.l2raw.txt
rm -f $rep.ncu-rep
