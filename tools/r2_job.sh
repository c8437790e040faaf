# usage: bash tools/r2_job.sh <tag> <command...>  — runs one command on the GPU box, output to gpurun_out/<tag>.log
tag=$1; shift
mkdir -p gpurun_out
( "$@" ) > gpurun_out/$tag.log 2>&1
echo "rc=$?" >> gpurun_out/$tag.log
tail -30 gpurun_out/$tag.log
