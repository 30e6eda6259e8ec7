for L in paper_1511_03296_b200/alt/libfbs_pre.so paper_1511_03296_b200/alt/libfbs_c3.so; do
FBS_PCG_GROUPS=1 FBS_LIB=$PWD/$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__registers_per_thread,launch__grid_size --clock-control none -k regex:"k_spmv2|k_tree_lift" -c 12 --csv python scripts/prof_pcg.py 6 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
rows=list(csv.reader([l for l in sys.stdin if l.startswith('\"')]))
h=rows[0]
for r in rows[1:]: print('$L'[-10:], r[h.index('Kernel Name')][:30], r[h.index('Metric Name')], r[h.index('Metric Value')])
"
done
