# knob sweep on the slowest workloads (run under gpurun); one JSON line per (knobs, cfg)
mkdir -p gpurun_out
C='[{"cfg":[26,4,"glex"]},{"cfg":[24,3,"grlex"]},{"cfg":[24,3,"glex"]},{"cfg":[26,4,"gray"]}]'
L='[{"cfg":[28,3,"lex"]}]'
run() { echo "== $*"; env "$@" timeout 120 python tools/sweep.py "$C"; }
runl() { echo "== L $*"; env "$@" timeout 60 python tools/sweep.py "$L"; }
{
run X=0
for t in 384 1024 1536; do run GC_TARGET_ACCEPTED=$t; done
for p in 512 2048; do run GC_PARTIAL_S=$p; done
for i in 1 2 8; do run GC_ITEMS_PER_WARP=$i; done
for b in 8 10 14; do run GC_SPLIT_BITS=$b; done
for g in 4096 65536; do run GC_GEO_HEAD=$g; done
runl X=0
for t in 256 512 768; do runl GC_TARGET_ACCEPTED=$t; done
for p in 256 1024; do runl GC_PARTIAL_S=$p; done
for b in 8 9 11; do runl GC_SPLIT_BITS=$b; done
for g in 8192 32768; do runl GC_GEO_HEAD=$g; done
for s in 65536 262144; do runl GC_SUB_MAX=$s; done
} > gpurun_out/sweep_knobs.log 2>&1
