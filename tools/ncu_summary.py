"""Summarise an .ncu-rep: key metrics, stall reasons and the SASS opcode mix."""
import csv, io, subprocess, sys
from collections import Counter

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'smsp__inst_executed.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'lts__t_bytes.sum',
        'sm__cycles_elapsed.avg.per_second']

def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

def main(rep, kernel_row=0):
    hdr, units, vals = raw(rep)
    v = vals[kernel_row]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k); print(f'{k:70s} {v[i]:>18s} {units[i]}')
    st = []
    for i, h in enumerate(hdr):
        if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
            try: st.append((float(v[i]), h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
            except ValueError: pass
    print('stalls per issue:', ', '.join(f'{n}={x:.2f}' for x, n in sorted(st, reverse=True)[:10]))
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]; data = rows[2:]
    isrc = h.index('Source'); iex = h.index('Instructions Executed'); iss = h.index('Warp Stall Sampling (All Samples)')
    ex = Counter(); stc = Counter()
    for r in data:
        toks = r[isrc].split()
        if not toks: continue
        op = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
        op = op.split('.')[0]
        ex[op] += int(r[iex] or 0); stc[op] += int(r[iss] or 0)
    te = sum(ex.values()) or 1; ts = sum(stc.values()) or 1
    print('opcode mix (exec%, stall%):', ', '.join(f'{o}={100*c/te:.1f}/{100*stc[o]/ts:.1f}' for o, c in ex.most_common(16)))

if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
