set -x
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config $CFG --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r20_${CFG}_$tag.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r20_${CFG}_$tag.json').read().strip().splitlines()[-1]);print('$CFG $tag', round(d['ms_per_step'],4))"; }
for CFG in c5 c4; do
  export CFG
  run base PLANC_B200_X=0
  run streams2 PLANC_B200_STREAMS=2
  run streams8 PLANC_B200_STREAMS=8
  run pdl0 PLANC_B200_PDL=0
  run occ2_0 PLANC_B200_OCC2=0
  run epi8_0 PLANC_B200_EPI8=0
  run splitk0 PLANC_B200_SPLITK=0
  run sync0 PLANC_B200_SYNC_EDGES=0
done
