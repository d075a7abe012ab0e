# Full measurement pass + summaries made ON the GPU box (the .ncu-rep files are
# too large to bring back); only the summaries return in gpurun_out/<tag>_prof.
# Usage: bash scripts/gpu_full_pass.sh <tag> <commit>   (the box has no .git: pass the commit)
TAG=${1:-r1}
COMMIT=${2:-unknown}
bash scripts/gpu_full.sh $TAG
python scripts/make_profiles.py $TAG $COMMIT > gpurun_out/$TAG/make_profiles.log 2>&1
mkdir -p gpurun_out/${TAG}_prof
cp profiles/${TAG}_* profiles/ncu_traffic.json gpurun_out/${TAG}_prof/ 2>/dev/null
rm -f gpurun_out/$TAG/*.ncu-rep
du -sh gpurun_out
