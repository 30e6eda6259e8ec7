"""Summarise an ncu --set full report, one block per profiled launch: time, DRAM bytes,
throughput, occupancy, top stall reasons."""
import csv
import json
import subprocess
import sys

KEYS = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block_dynamic',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_warps',
        'sm__maximum_warps_per_active_cycle_pct', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum']


def summary(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    H, U = r[0], r[1]
    outs = []
    for V in r[2:]:
        out = {k: V[H.index(k)] + ((' ' + U[H.index(k)]) if U[H.index(k)] else '') for k in KEYS if k in H}
        stalls = {}
        for i, name in enumerate(H):
            if name.startswith('smsp__pcsamp_warps_issue_stalled_') and not name.endswith('not_issued'):
                try:
                    stalls[name.replace('smsp__pcsamp_warps_issue_stalled_', '')] = float(V[i].replace(',', ''))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        out['stall_top'] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        outs.append(out)
    return outs


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(p)
        print(json.dumps(summary(p), indent=1))
