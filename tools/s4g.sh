bash tools/odsab.sh s4g imagenet1k 4 base fast2 fast4 fast3
