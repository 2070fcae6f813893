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
    if (m < INT64_C(7168)) {
        if (n < INT64_C(1620)) {
            if (m < INT64_C(113)) {
                if (m < INT64_C(80)) {
                    if (n < INT64_C(702)) {
                        if (n < INT64_C(227)) {
                            if (m < INT64_C(57)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(2897)) {
                            if (m < INT64_C(29)) {
                                if (k < INT64_C(1620)) {
                                    if (m < INT64_C(2)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(6)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(12)) {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(3)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(8)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(6)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(12)) {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(227)) {
                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(992)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(1449)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(1268)) {
                    if (k < INT64_C(136)) {
                        if (m < INT64_C(555)) {
                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(544)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(992)) {
                            if (n < INT64_C(111)) {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(272)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(272)) {
                                        if (m < INT64_C(555)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(555)) {
                                            if (k < INT64_C(471)) {
                                                if (n < INT64_C(79)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(448)) {
                                    if (n < INT64_C(203)) {
                                        if (k < INT64_C(744)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (n < INT64_C(405)) {
                                            if (m < INT64_C(317)) {
                                                if (m < INT64_C(225)) {
                                                    if (k < INT64_C(1536)) {
                                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(1449)) {
                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(3072)) {
                                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (k < INT64_C(405)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(2173)) {
                                                        select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(203)) {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(363)) {
                                            if (k < INT64_C(1087)) {
                                                if (k < INT64_C(744)) {
                                                    if (n < INT64_C(144)) {
                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(634)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(512)) {
                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(1449)) {
                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(3072)) {
                                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(405)) {
                                if (m < INT64_C(278)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(555)) {
                                        if (k < INT64_C(287)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(287)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(167)) {
                        if (k < INT64_C(444)) {
                            if (n < INT64_C(46)) {
                                if (m < INT64_C(2218)) {
                                    select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(118)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(4435)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(167)) {
                                                if (n < INT64_C(28)) {
                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(2218)) {
                                    if (k < INT64_C(222)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(314)) {
                                        if (m < INT64_C(4435)) {
                                            if (k < INT64_C(68)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(222)) {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (n < INT64_C(91)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(768)) {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(815)) {
                                    if (n < INT64_C(79)) {
                                        if (m < INT64_C(4435)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(4435)) {
                            if (n < INT64_C(768)) {
                                if (m < INT64_C(2218)) {
                                    if (k < INT64_C(111)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(182)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(363)) {
                                                if (k < INT64_C(725)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(1536)) {
                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(363)) {
                                        if (k < INT64_C(1630)) {
                                            if (k < INT64_C(182)) {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(725)) {
                                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(111)) {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(1087)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(64)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(1630)) {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(363)) {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(10138)) {
                if (m < INT64_C(1268)) {
                    if (m < INT64_C(278)) {
                        if (m < INT64_C(12)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(725)) {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(40)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                if (m < INT64_C(3)) {
                    select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                } else {
                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (n < INT64_C(46)) {
            if (k < INT64_C(118)) {
                if (m < INT64_C(70960)) {
                    if (m < INT64_C(17740)) {
                        if (k < INT64_C(56)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(35480)) {
                            if (k < INT64_C(56)) {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(56)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(141920)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(35480)) {
                    if (k < INT64_C(167)) {
                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                    return out;
                }
            }
        } else {
            if (k < INT64_C(815)) {
                if (m < INT64_C(17740)) {
                    if (n < INT64_C(111)) {
                        if (k < INT64_C(97)) {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(194)) {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(111)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(70960)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(35480)) {
                    if (k < INT64_C(1630)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_BF16_NN_H */
