#ifndef SELECT_BF16_NN_H
#define SELECT_BF16_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nn_config;

static inline select_bf16_nn_config select_bf16_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(1087)) {
        if (m < INT64_C(35480)) {
            if (m < INT64_C(634)) {
                if (n < INT64_C(444)) {
                    if (n < INT64_C(144)) {
                        if (m < INT64_C(278)) {
                            if (m < INT64_C(159)) {
                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(139)) {
                            if (n < INT64_C(227)) {
                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(287)) {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(248)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(1145)) {
                        if (k < INT64_C(363)) {
                            if (m < INT64_C(278)) {
                                if (m < INT64_C(139)) {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(124)) {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(725)) {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(725)) {
                                if (m < INT64_C(70)) {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (n < INT64_C(351)) {
                    if (m < INT64_C(2218)) {
                        if (n < INT64_C(46)) {
                            if (m < INT64_C(1109)) {
                                select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(167)) {
                                    select_bf16_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                if (n < INT64_C(111)) {
                                    if (k < INT64_C(272)) {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(79)) {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(287)) {
                                    if (k < INT64_C(992)) {
                                        if (m < INT64_C(1109)) {
                                            if (k < INT64_C(744)) {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(136)) {
                            if (k < INT64_C(79)) {
                                if (m < INT64_C(17740)) {
                                    if (m < INT64_C(4435)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(46)) {
                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(8870)) {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {8u, 2u, 8u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(21)) {
                                        select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(111)) {
                                    if (k < INT64_C(168)) {
                                        if (n < INT64_C(28)) {
                                            if (m < INT64_C(4435)) {
                                                if (k < INT64_C(118)) {
                                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(8870)) {
                                                    if (k < INT64_C(118)) {
                                                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (m < INT64_C(17740)) {
                                                        if (k < INT64_C(118)) {
                                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(17740)) {
                                                if (m < INT64_C(4435)) {
                                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(146)) {
                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            if (k < INT64_C(471)) {
                                                if (m < INT64_C(4435)) {
                                                    if (k < INT64_C(272)) {
                                                        if (n < INT64_C(46)) {
                                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        if (n < INT64_C(79)) {
                                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                } else {
                                                    if (k < INT64_C(222)) {
                                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(222)) {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(4435)) {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            if (k < INT64_C(363)) {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(363)) {
                                                select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(544)) {
                                                    select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(17740)) {
                                if (k < INT64_C(28)) {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(182)) {
                                        if (m < INT64_C(4435)) {
                                            select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(46)) {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(40)) {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(111)) {
                            if (k < INT64_C(79)) {
                                select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(1109)) {
                                if (n < INT64_C(702)) {
                                    if (k < INT64_C(182)) {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(405)) {
                                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(725)) {
                                            select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(111)) {
                                select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(4435)) {
                                    if (n < INT64_C(725)) {
                                        if (k < INT64_C(182)) {
                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(111)) {
                if (n < INT64_C(46)) {
                    if (n < INT64_C(20)) {
                        select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(21)) {
                        select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                        return out;
                    } else {
                        if (m < INT64_C(70960)) {
                            if (k < INT64_C(97)) {
                                select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                select_bf16_nn_config out = {8u, 2u, 8u, 16u, 16u};
                return out;
            }
        }
    } else {
        if (m < INT64_C(3584)) {
            if (k < INT64_C(10753)) {
                if (m < INT64_C(1109)) {
                    if (k < INT64_C(4345)) {
                        if (n < INT64_C(2024)) {
                            if (m < INT64_C(3)) {
                                if (k < INT64_C(1620)) {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(2897)) {
                                        select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(3072)) {
                                    if (m < INT64_C(12)) {
                                        if (m < INT64_C(6)) {
                                            if (k < INT64_C(1620)) {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(278)) {
                                            if (m < INT64_C(40)) {
                                                if (k < INT64_C(1620)) {
                                                    select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(2173)) {
                                                        select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(555)) {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(2173)) {
                                                    select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (n < INT64_C(363)) {
                                                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(2)) {
                                select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(8)) {
                                    select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(139)) {
                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(393)) {
                                select_bf16_nn_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(1537)) {
                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(2509)) {
                            if (m < INT64_C(2535)) {
                                if (n < INT64_C(363)) {
                                    select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(363)) {
                                    select_bf16_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_nn_config out = {8u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                select_bf16_nn_config out = {2u, 1u, 8u, 8u, 8u};
                return out;
            }
        } else {
            if (k < INT64_C(1630)) {
                if (m < INT64_C(35480)) {
                    if (m < INT64_C(17740)) {
                        if (m < INT64_C(8870)) {
                            if (n < INT64_C(182)) {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(182)) {
                                select_bf16_nn_config out = {2u, 1u, 4u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {8u, 2u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {4u, 1u, 4u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_bf16_nn_config out = {8u, 2u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                if (n < INT64_C(363)) {
                    if (m < INT64_C(8870)) {
                        select_bf16_nn_config out = {2u, 1u, 8u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_bf16_nn_config out = {8u, 2u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_BF16_NN_H */
