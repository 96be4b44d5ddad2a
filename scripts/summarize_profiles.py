"""Summarise ncu reports into profiles/ (tracked):
    python scripts/summarize_profiles.py ROUND CONFIG REPORT OBJ SRC KERNEL_SUBSTR "command" [CONFIG REPORT ...]
Writes profiles/<CONFIG>_dram_per_launch.json (bench.py roofline.traffic),
profiles/<ROUND>_ncu_<CONFIG>.md (metrics + hot source lines) and merges the
raw metrics into profiles/<ROUND>_ncu_raw_metrics.json."""
import csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, 'scripts'))
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__average_warp_latency_per_inst_issued.ratio',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__shared_mem_per_block_dynamic', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct', 'smsp__inst_executed.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (v[h.index(k)], u[h.index(k)]) for k in KEYS + ['Kernel Name'] if k in h}


def to_bytes(val, unit):
    f = float(val)
    return f * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'Tbyte': 1e12}.get(unit, 1)


def main():
    rnd = sys.argv[1]
    args = sys.argv[2:]
    rawp = os.path.join(ROOT, 'profiles', f'{rnd}_ncu_raw_metrics.json')
    allraw = json.load(open(rawp)) if os.path.exists(rawp) else {}
    while args:
        cfg, rep, obj, src, ksub, cmd = args[:6]
        args = args[6:]
        m = raw(rep)
        dram = to_bytes(*m['dram__bytes_read.sum']) + to_bytes(*m['dram__bytes_write.sum'])
        json.dump({'dram_bytes_per_launch': dram, 'kernel': m['Kernel Name'][0],
                   'source': f'ncu --set full, one launch of: {cmd} ({rnd})'},
                  open(os.path.join(ROOT, 'profiles', f'{cfg}_dram_per_launch.json'), 'w'), indent=1)
        allraw[cfg] = {'command': cmd, 'metrics': {k: list(v) for k, v in m.items()}}
        sass = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                              capture_output=True, text=True).stdout
        tmp = f'/tmp/{cfg}_sass.csv'
        open(tmp, 'w').write(sass)
        lines = subprocess.run([sys.executable, os.path.join(ROOT, 'scripts', 'sass_lines.py'), obj, ksub, tmp, src, '20'],
                               capture_output=True, text=True).stdout
        with open(os.path.join(ROOT, 'profiles', f'{rnd}_ncu_{cfg}.md'), 'w') as f:
            f.write(f'# {cfg}: ncu --set full ({rnd})\n\nCommand: `{cmd}`\n\n| metric | unit | value |\n|---|---|---|\n')
            for k, (v, u) in m.items():
                f.write(f'| {k} | {u} | {v} |\n')
            f.write(f'\nDRAM bytes per launch (read + write): {dram:.4g}\n\n')
            f.write('## Stall samples / executed instructions by source function and line\n'
                    '(scripts/sass_lines.py: SASS page joined with nvdisasm line info)\n\n```\n' + lines + '```\n')
        print(cfg, m['gpu__time_duration.sum'], f'dram {dram:.3g}')
    json.dump(allraw, open(rawp, 'w'), indent=1)


if __name__ == '__main__':
    main()
