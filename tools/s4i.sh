bash tools/odsab.sh s4i imagenet1k 4 base sigw
