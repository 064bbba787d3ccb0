# Round evidence beyond prof_round.sh (run under gpurun): config sweep, panel sweeps / phase profiles, scaling
# models, exposed swap time, QR line.  Usage: bash tools/round_evidence.sh r06
R=${1:-r06}
mkdir -p gpurun_out
set -x
python tools/config_sweep.py gpurun_out/${R}_configs.json > gpurun_out/${R}_configs.log 2>&1
{ python tools/panel_sweep.py --m 32768,24576,16384,12288,8192,4096,2048,1024 --kernel 0,1,2,4 --tag auto-split;
  PFLU_AUTO_REC_LEAF=0 python tools/panel_sweep.py --m 32768,16384,8192,4096,2048 --kernel 1,2 --tag no-split;
  PFLU_AUTO_REC_LEAF=0 PFLU_PANEL_V2=0 python tools/panel_sweep.py --m 32768,16384,8192,4096,2048,1024 --kernel 2 --tag v1-cluster-no-split;
  python tools/panel_sweep.py --m 8192,4096,2048,1024,512 --w 128 --kernel 2 --tag w128; } > gpurun_out/${R}_panel_sweep.log 2>&1
{ for M in 2048 8192; do PFLU_LIB_PATH=tools/libpflu_prof.so python tools/panel_prof.py $M 256 0 0 0 2; done;
  PFLU_LIB_PATH=tools/libpflu_prof.so python tools/panel_prof.py 32768 128 0 0 0 4; } > gpurun_out/${R}_panel_prof.log 2>&1
python tools/emu_scaling.py --ranks 1,2,4,8 --driver cpp > gpurun_out/${R}_emu_scaling_cpp.jsonl 2>&1
python tools/emu_scaling.py --ranks 1,2,4,8 --driver dist > gpurun_out/${R}_emu_scaling_dist.jsonl 2>&1
{ python tools/exposed_swap.py; PFLU_EMU_RANKS=8 python tools/chain_gaps.py; } > gpurun_out/${R}_chain.log 2>&1
python bench.py --kind qr --e2e-steps 1 > gpurun_out/${R}_qr_bench_line.jsonl 2> gpurun_out/${R}_qr_bench.err
tail -1 gpurun_out/${R}_qr_bench_line.jsonl
