"""Summarise an .ncu-rep (raw page) into the handful of numbers we track.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [more.ncu-rep ...]"""
import csv, io, subprocess, sys
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_bytes.sum', 'l1tex__t_bytes.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__grid_size',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts.sum', 'l1tex__lsu_writeback_active.sum',
        'l1tex__m_xbar2l1tex_read_bytes.sum', 'l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__cycles_elapsed.avg', 'sm__cycles_elapsed.avg.per_second',
        'lts__cycles_elapsed.avg.per_second', 'sm__inst_executed_pipe_lsu.sum',
        'smsp__thread_inst_executed_per_inst_executed.ratio',
        'lts__t_sectors_op_read.sum', 'lts__t_sectors_op_write.sum',
        'lts__average_t_sector_hit_rate_srcunit_tex_realtime.pct',
        'l1tex__m_xbar2l1tex_read_sectors.sum']
for path in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"== {path} :: {vals[hdr.index('Kernel Name')][:80] if 'Kernel Name' in hdr else ''}")
        for i, h in enumerate(hdr):
            if h in WANT or ('issue_stalled' in h and h.endswith('per_issue_active.ratio') and float(vals[i] or 0) > 0.2):
                print(f"  {h:86s} {units[i]:14s} {vals[i]}")
