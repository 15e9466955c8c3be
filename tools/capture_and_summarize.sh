# usage: capture_and_summarize.sh TAG "model system" ... — capture (capture_profiles.sh), summarise
# into profiles/round2/<model>_<system>/ on the box (launch shares + DRAM traffic JSON read by
# bench.py), keep only small artefacts in gpurun_out/
TAG=$1
bash tools/capture_profiles.sh "$@"
shift
for cfg in "$@"; do
  set -- $cfg
  python tools/profile_summary.py round2/$1_$2 gpurun_out/launches_${TAG}_$1_$2.csv gpurun_out/full_${TAG}_$1_$2.ncu-rep $1 $2
  mkdir -p gpurun_out/profiles/round2/$1_$2
  cp profiles/round2/$1_$2/*.md gpurun_out/profiles/round2/$1_$2/
done
cp profiles/round2/*.json gpurun_out/profiles/round2/
rm -f gpurun_out/full_${TAG}_*.ncu-rep
