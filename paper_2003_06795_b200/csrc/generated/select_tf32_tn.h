#ifndef SELECT_TF32_TN_H
#define SELECT_TF32_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tn_config;

static inline select_tf32_tn_config select_tf32_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(992)) {
        if (m < INT64_C(35480)) {
            if (m < INT64_C(448)) {
                if (k < INT64_C(351)) {
                    if (k < INT64_C(79)) {
                        if (m < INT64_C(113)) {
                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(79)) {
                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(287)) {
                            if (k < INT64_C(444)) {
                                if (m < INT64_C(278)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                if (m < INT64_C(70)) {
                                    if (k < INT64_C(702)) {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(702)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(702)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(136)) {
                    if (k < INT64_C(30)) {
                        if (m < INT64_C(17740)) {
                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(21)) {
                                select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(46)) {
                            if (k < INT64_C(167)) {
                                if (m < INT64_C(4435)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(118)) {
                                        if (k < INT64_C(56)) {
                                            if (m < INT64_C(17740)) {
                                                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            if (n < INT64_C(28)) {
                                                select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(17740)) {
                                                if (n < INT64_C(28)) {
                                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(2218)) {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(4435)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(17740)) {
                                if (k < INT64_C(544)) {
                                    if (m < INT64_C(8870)) {
                                        if (k < INT64_C(222)) {
                                            if (m < INT64_C(1568)) {
                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(4435)) {
                                                    if (k < INT64_C(111)) {
                                                        select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (n < INT64_C(79)) {
                                                if (m < INT64_C(1109)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(2218)) {
                                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(4435)) {
                                                            select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(4435)) {
                                                    if (k < INT64_C(444)) {
                                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(1109)) {
                                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (m < INT64_C(2218)) {
                                                                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    }
                                                } else {
                                                    if (k < INT64_C(363)) {
                                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    } else {
                                        if (n < INT64_C(91)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(4435)) {
                                            if (m < INT64_C(2218)) {
                                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(8870)) {
                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (n < INT64_C(91)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            } else {
                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(405)) {
                        if (m < INT64_C(2218)) {
                            if (k < INT64_C(111)) {
                                if (m < INT64_C(1109)) {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(702)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1109)) {
                                        if (k < INT64_C(227)) {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(46)) {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(28)) {
                                        if (m < INT64_C(4435)) {
                                            select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(4435)) {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(8870)) {
                                                select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {8u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(544)) {
                                    if (m < INT64_C(4435)) {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(17740)) {
                                            if (k < INT64_C(182)) {
                                                if (k < INT64_C(91)) {
                                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {8u, 1u, 8u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(8870)) {
                                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(157)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (n < INT64_C(203)) {
                                select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (n < INT64_C(512)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(118)) {
                if (n < INT64_C(118)) {
                    if (m < INT64_C(567677)) {
                        select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(40)) {
                        select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_tn_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(91)) {
                    if (k < INT64_C(146)) {
                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(194)) {
                            if (m < INT64_C(100352)) {
                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(2173)) {
            if (m < INT64_C(3)) {
                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                return out;
            } else {
                if (m < INT64_C(1792)) {
                    if (m < INT64_C(1109)) {
                        if (k < INT64_C(1620)) {
                            if (n < INT64_C(716)) {
                                if (m < INT64_C(555)) {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(363)) {
                                                select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(393)) {
                                    if (m < INT64_C(28)) {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(70)) {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(12)) {
                                select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    if (m < INT64_C(40)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(182)) {
                        if (m < INT64_C(35480)) {
                            if (m < INT64_C(8870)) {
                                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(17740)) {
                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(70960)) {
                                select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(141920)) {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(2535)) {
                            select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                select_tf32_tn_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(3584)) {
                if (n < INT64_C(3548)) {
                    if (m < INT64_C(393)) {
                        if (m < INT64_C(12)) {
                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(4345)) {
                                if (m < INT64_C(56)) {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(139)) {
                                    select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(1255)) {
                            if (m < INT64_C(1109)) {
                                if (n < INT64_C(363)) {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {8u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    select_tf32_tn_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                if (k < INT64_C(7095)) {
                    if (n < INT64_C(363)) {
                        if (m < INT64_C(8870)) {
                            select_tf32_tn_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_TF32_TN_H */
